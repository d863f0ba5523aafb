// mpk.cu -- matrix-powers kernel: [v, A v, ..., A^J v] of v = src * scale for the 5-point
// (2D) and 7-point (3D) stencils in one pass over src, with a width-J ghost zone.
//
// Replaces krylov_block (block.hpp:59-67) / krylov_pair (sstep.hpp:71-81): each power is
// bit-identical to J successive reference spmv calls (sparse.hpp:135-146) because every
// stencil point is evaluated in the reference's ascending-column order with separately
// rounded multiplies and adds; out-of-domain neighbours enter as exact zeros, which leaves
// the sum's bits unchanged (adding +-0.0 to a sum that starts at +0.0).
//
// 2D: a CTA owns an output strip of W columns x R rows and streams it in y.  Each thread owns
// one column of the strip extended by J on both sides; level j keeps its last three rows in
// registers (the y-neighbours) and its newest row in a double-buffered shared-memory line
// (the x-neighbours).  Level j at step t produces row t-j, so one __syncthreads per row step
// advances all J levels.  3D works the same with an (x,y) tile streamed in z.
//
// Optionally the kernel fuses the products X_l . (A^j v) of the produced powers with up to
// MPK_MAXX extra vectors (the first block-MGS round of s-step Arnoldi, sstep.hpp:341),
// written as deterministic per-CTA partials.
#include <algorithm>
#include <cstring>

#include "device_util.cuh"
#include "skc_internal.hpp"

namespace skc {

namespace {

constexpr int MPK_MAXJ = 8;
constexpr int MPK_MAXX = 8;

struct MpkDesc {
  DevOp op;
  const double* src;
  const double* scale;  // device scalar or nullptr
  double* out[MPK_MAXJ + 1];
  int J;
  // tiles
  int W, R;        // 2D: output strip width, rows per CTA; 3D: W = tile x, R = tile y, Z = planes per CTA
  int Z;
  int tiles_x, tiles_y;
  // fused products
  int nx_dots;  // number of extra vectors (0 = none)
  const double* X[MPK_MAXX];
  int jdot0;  // products with levels jdot0..J
  double* partials;
  int dot0, G;
  const int* halt;
  const int* cond;
};

// coefficient of slot t at point p (row-major neighbour order -z,-y,-x,C,+x,+y,+z)
template <int DIM, int KIND>
__device__ __forceinline__ void coefs(const DevOp& op, int64_t p, const bool (&pres)[7], const int64_t (&nb)[7],
                                      double (&val)[7]) {
  if (KIND == kStencilConst) {
#pragma unroll
    for (int t = 0; t < 7; ++t) val[t] = op.coef[t];
  } else if (KIND == kStencilDia) {
#pragma unroll
    for (int t = 0; t < 7; ++t) val[t] = (DIM == 2 && (t == 0 || t == 6)) ? 0.0 : op.dia[t * op.n + p];
  } else {
    const double kp = op.kcell[p];
    double d = 0.0;
    bool first = true;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
      if (t == 3) continue;
      if (DIM == 2 && (t == 0 || t == 6)) continue;
      const double kq = pres[t] ? op.kcell[nb[t]] : kp;
      const double kf = pres[t] ? __ddiv_rn(__dmul_rn(__dmul_rn(2.0, kp), kq), __dadd_rn(kp, kq)) : kp;
      d = first ? kf : __dadd_rn(d, kf);
      first = false;
      val[t] = t < 3 ? __dsub_rn(-kf, op.ch2) : __dadd_rn(-kf, op.ch2);
    }
    val[3] = d;
  }
}

// ------------------------------------------------------------------ 2D
template <int KIND, int J, bool DOTS>
__global__ void __launch_bounds__(288) k_mpk2d(const __grid_constant__ MpkDesc d) {
  if (skip_launch(d.halt, d.cond)) return;
  __shared__ double line[J][2][288];  // level j's newest row, double-buffered by step parity
  const int tid = threadIdx.x;
  const int nx = (int)d.op.nx, ny = (int)d.op.ny;
  const int tx = blockIdx.x % d.tiles_x, ty = blockIdx.x / d.tiles_x;
  const int x0 = tx * d.W, y0 = ty * d.R;
  const int y1 = min(ny, y0 + d.R);
  const int c = x0 - J + tid;  // this thread's column
  const bool colin = c >= 0 && c < nx && tid < d.W + 2 * J;
  const bool outcol = tid >= J && tid < J + d.W && c < nx;
  const bool hasW = c > 0, hasE = c + 1 < nx;
  const double scale = d.scale ? *d.scale : 1.0;
  double* outs[J + 1];
#pragma unroll
  for (int j = 0; j <= J; ++j) outs[j] = d.out[j];
  double win[J + 1][3];  // per level: rows (r-1, r, r+1) around the row the next level computes
#pragma unroll
  for (int j = 0; j <= J; ++j) win[j][0] = win[j][1] = win[j][2] = 0.0;
  // fused products: the J+1 extra vectors X_l against every produced level 1..J
  constexpr int NX = J + 1;
  constexpr int NACC = DOTS ? NX * J : 1;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  // slab geometry: local row t is global row row0 + t; rows just outside the slab come from
  // the halo buffers (filled by the exchange), rows outside the grid are Dirichlet zeros
  const int64_t row0 = d.op.row0, rows_g = d.op.rows_global;
  const int H = (int)d.op.halo_rows;
  auto fetch = [&](int t) -> double {
    const int64_t tg = row0 + t;
    if (!colin || tg < 0 || tg >= rows_g || t < y0 - J || t >= y1 + J) return 0.0;
    const double* rowp = t < 0 ? d.op.hlo + (int64_t)(t + H) * nx
                               : (t >= ny ? d.op.hhi + (int64_t)(t - ny) * nx : d.src + (int64_t)t * nx);
    return rowp[c];
  };

  // level-0 rows are prefetched PF steps ahead so each thread keeps PF loads in flight
  constexpr int PF = 8;
  double pf[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) pf[k] = fetch(y0 - J + k);
  for (int t = y0 - J; t < y1 + J; ++t) {
    const int par = t & 1;
    // level 0: row t
    const double s0 = pf[0];
#pragma unroll
    for (int k = 0; k + 1 < PF; ++k) pf[k] = pf[k + 1];
    pf[PF - 1] = fetch(t + PF);
    double v0 = 0.0;
    if (colin && row0 + t >= 0 && row0 + t < rows_g) v0 = d.scale ? __dmul_rn(s0, scale) : s0;
    win[0][0] = win[0][1];
    win[0][1] = win[0][2];
    win[0][2] = v0;
    line[0][par][tid] = v0;
    if (outs[0] && outcol && t >= y0 && t < y1) outs[0][(int64_t)t * nx + c] = v0;
    // levels 1..J: level j computes row r = t - j
#pragma unroll
    for (int j = 1; j <= J; ++j) {
      const int r = t - j;
      const int64_t rg = row0 + r;
      double v = 0.0;
      // level j is needed (and its inputs valid) only within J-j rows of the CTA's rows
      if (colin && rg >= 0 && rg < rows_g && r >= y0 - (J - j) && r < y1 + (J - j)) {
        // x-neighbours of level j-1 at row r: its line written one step ago
        const double* ln = line[j - 1][par ^ 1];
        // (tile-edge threads see a zero instead of the neighbour: they are ghost columns whose
        // values never reach an output)
        const double xw = (hasW && tid > 0) ? ln[tid - 1] : 0.0;
        const double xe = (hasE && tid + 1 < 288) ? ln[tid + 1] : 0.0;
        const double ys = rg > 0 ? win[j - 1][0] : 0.0;
        const double yn = rg + 1 < rows_g ? win[j - 1][2] : 0.0;
        double cS, cW, cC, cE, cN;
        if (KIND == kStencilConst) {
          cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
        } else {
          bool pres[7];
          int64_t nb[7];
          const int64_t p = (int64_t)r * nx + c;
          pres[0] = pres[6] = false;
          pres[1] = rg > 0;
          pres[2] = hasW;
          pres[3] = true;
          pres[4] = hasE;
          pres[5] = rg + 1 < rows_g;
          nb[0] = nb[6] = nb[3] = p;
          nb[1] = p - nx;
          nb[2] = p - 1;
          nb[4] = p + 1;
          nb[5] = p + nx;
          double val[7];
          coefs<2, KIND>(d.op, p, pres, nb, val);
          cS = val[1], cW = val[2], cC = val[3], cE = val[4], cN = val[5];
        }
        // S, W, C, E, N (ascending column); absent neighbours are exact zeros
        double a = 0.0;
        a = __dadd_rn(a, __dmul_rn(cS, ys));
        a = __dadd_rn(a, __dmul_rn(cW, xw));
        a = __dadd_rn(a, __dmul_rn(cC, win[j - 1][1]));
        a = __dadd_rn(a, __dmul_rn(cE, xe));
        a = __dadd_rn(a, __dmul_rn(cN, yn));
        v = a;
      }
      win[j][0] = win[j][1];
      win[j][1] = win[j][2];
      win[j][2] = v;
      if (j < J) line[j < J ? j : 0][par][tid] = v;
      if (outcol && r >= y0 && r < y1) {
        const int64_t p = (int64_t)r * nx + c;
        if (outs[j]) outs[j][p] = v;
        if (DOTS) {
#pragma unroll
          for (int x = 0; x < NX; ++x) acc[x * J + (j - 1)] = fma(d.X[x][p], v, acc[x * J + (j - 1)]);
        }
      }
    }
    __syncthreads();
  }
  if (DOTS) {
    // fixed-order CTA reduction: product (x, level j) -> dot0 + x*J + (j-1)
    __shared__ double red[9][NACC];
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) red[warp][q] = v;
    }
    __syncthreads();
    for (int e = tid; e < NACC; e += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < 9; ++w) s += red[w][e];
      d.partials[(int64_t)(d.dot0 + e) * kPartialPitch + blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------ 3D
// tile: TXe x TYe threads (extended by J each side), streamed over d.Z planes
template <int KIND, int J, int TXE, int TYE, bool DOTS>
__global__ void __launch_bounds__(TXE* TYE) k_mpk3d(const __grid_constant__ MpkDesc d) {
  if (skip_launch(d.halt, d.cond)) return;
  __shared__ double plane[J][2][TYE][TXE];
  const int lx = threadIdx.x % TXE, ly = threadIdx.x / TXE;
  const int64_t nx = d.op.nx, ny = d.op.ny, nz = d.op.nz;
  const int64_t pl = nx * ny;
  const int ntile = d.tiles_x * d.tiles_y;
  const int tile = blockIdx.x % ntile, zc = blockIdx.x / ntile;
  const int tx = tile % d.tiles_x, ty = tile / d.tiles_x;
  const int64_t x = (int64_t)tx * d.W - J + lx, y = (int64_t)ty * d.R - J + ly;
  const int64_t z0 = (int64_t)zc * d.Z, z1 = min(nz, z0 + d.Z);
  const bool in = x >= 0 && x < nx && y >= 0 && y < ny;
  const bool outp = lx >= J && lx < J + d.W && ly >= J && ly < J + d.R && x < nx && y < ny;
  const double scale = d.scale ? *d.scale : 1.0;
  double win[J + 1][3];
#pragma unroll
  for (int j = 0; j <= J; ++j) win[j][0] = win[j][1] = win[j][2] = 0.0;
  constexpr int NACC = DOTS ? (J + 1) * J : 1;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;

  // z-slab geometry (see the 2D kernel): plane t is global plane row0 + t
  const int64_t row0 = d.op.row0, rows_g = d.op.rows_global;
  const int64_t H = d.op.halo_rows;
  const int64_t xy = y * nx + x;
  auto fetch = [&](int64_t t) -> double {
    const int64_t tg = row0 + t;
    if (!in || tg < 0 || tg >= rows_g || t < z0 - J || t >= z1 + J) return 0.0;
    const double* pp =
        t < 0 ? d.op.hlo + (t + H) * pl : (t >= nz ? d.op.hhi + (t - nz) * pl : d.src + t * pl);
    return pp[xy];
  };
  constexpr int PF = 4;
  double pf[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) pf[k] = fetch(z0 - J + k);
  for (int64_t t = z0 - J; t < z1 + J; ++t) {
    const int par = (int)(t & 1);
    const double s0 = pf[0];
#pragma unroll
    for (int k = 0; k + 1 < PF; ++k) pf[k] = pf[k + 1];
    pf[PF - 1] = fetch(t + PF);
    double v0 = 0.0;
    if (in && row0 + t >= 0 && row0 + t < rows_g) v0 = d.scale ? __dmul_rn(s0, scale) : s0;
    win[0][0] = win[0][1];
    win[0][1] = win[0][2];
    win[0][2] = v0;
    plane[0][par][ly][lx] = v0;
    if (d.out[0] && outp && t >= z0 && t < z1) d.out[0][t * pl + y * nx + x] = v0;
#pragma unroll
    for (int j = 1; j <= J; ++j) {
      const int64_t r = t - j;  // plane computed by level j
      const int64_t rg = row0 + r;
      double v = 0.0;
      if (in && rg >= 0 && rg < rows_g && r >= z0 - (J - j) && r < z1 + (J - j)) {
        const auto& P = plane[j - 1][par ^ 1];
        const double ys = ly > 0 ? P[ly - 1][lx] : 0.0;
        const double xw = lx > 0 ? P[ly][lx - 1] : 0.0;
        const double xe = lx + 1 < TXE ? P[ly][lx + 1] : 0.0;
        const double yn = ly + 1 < TYE ? P[ly + 1][lx] : 0.0;
        bool pres[7];
        int64_t nb[7];
        const int64_t p = r * pl + y * nx + x;
        pres[0] = rg > 0;
        pres[1] = y > 0;
        pres[2] = x > 0;
        pres[3] = true;
        pres[4] = x + 1 < nx;
        pres[5] = y + 1 < ny;
        pres[6] = rg + 1 < rows_g;
        nb[0] = p - pl;
        nb[1] = p - nx;
        nb[2] = p - 1;
        nb[3] = p;
        nb[4] = p + 1;
        nb[5] = p + nx;
        nb[6] = p + pl;
        double val[7];
        coefs<3, KIND>(d.op, p, pres, nb, val);
        double a = 0.0;
        a = __dadd_rn(a, __dmul_rn(val[0], pres[0] ? win[j - 1][0] : 0.0));
        a = __dadd_rn(a, __dmul_rn(val[1], pres[1] ? ys : 0.0));
        a = __dadd_rn(a, __dmul_rn(val[2], pres[2] ? xw : 0.0));
        a = __dadd_rn(a, __dmul_rn(val[3], win[j - 1][1]));
        a = __dadd_rn(a, __dmul_rn(val[4], pres[4] ? xe : 0.0));
        a = __dadd_rn(a, __dmul_rn(val[5], pres[5] ? yn : 0.0));
        a = __dadd_rn(a, __dmul_rn(val[6], pres[6] ? win[j - 1][2] : 0.0));
        v = a;
      }
      win[j][0] = win[j][1];
      win[j][1] = win[j][2];
      win[j][2] = v;
      if (j < J) plane[j < J ? j : 0][par][ly][lx] = v;
      if (outp && r >= z0 && r < z1) {
        const int64_t p = r * pl + y * nx + x;
        if (d.out[j]) d.out[j][p] = v;
        if (DOTS) {
#pragma unroll
          for (int q = 0; q < J + 1; ++q) acc[q * J + (j - 1)] = fma(d.X[q][p], v, acc[q * J + (j - 1)]);
        }
      }
    }
    __syncthreads();
  }
  if (DOTS) {
    constexpr int NW = TXE * TYE / 32;
    __shared__ double red[NW][NACC];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) red[warp][q] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < NACC; e += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += red[w][e];
      d.partials[(int64_t)(d.dot0 + e) * kPartialPitch + blockIdx.x] = s;
    }
  }
}

template <int KIND, int J>
void launch2d(Ctx& c, MpkDesc& d) {
  const int64_t nx = d.op.nx, ny = d.op.ny;
  d.W = (int)std::min<int64_t>(nx, 288 - 2 * J);
  d.tiles_x = (int)((nx + d.W - 1) / d.W);
  // rows per CTA: aim for ~2 CTAs per SM, at least 4J rows to bound the ghost-row overhead
  const int64_t target = 2LL * c.sm_count;
  int64_t R = std::max<int64_t>(4 * J, (ny * d.tiles_x + target - 1) / target);
  R = std::min<int64_t>(R, ny);
  d.R = (int)R;
  d.tiles_y = (int)((ny + R - 1) / R);
  d.G = d.tiles_x * d.tiles_y;
  if (d.nx_dots)
    k_mpk2d<KIND, J, true><<<d.G, 288, 0, c.stream>>>(d);
  else
    k_mpk2d<KIND, J, false><<<d.G, 288, 0, c.stream>>>(d);
}

template <int KIND, int J>
void launch3d(Ctx& c, MpkDesc& d) {
  constexpr int TXE = 32, TYE = 16;
  const int64_t nx = d.op.nx, ny = d.op.ny, nz = d.op.nz;
  d.W = TXE - 2 * J;
  d.R = TYE - 2 * J;
  d.tiles_x = (int)((nx + d.W - 1) / d.W);
  d.tiles_y = (int)((ny + d.R - 1) / d.R);
  const int64_t ntile = (int64_t)d.tiles_x * d.tiles_y;
  const int64_t target = 4LL * c.sm_count;
  int64_t zc = std::max<int64_t>(1, std::min<int64_t>(nz, target / std::max<int64_t>(1, ntile)));
  int64_t Z = std::max<int64_t>((nz + zc - 1) / zc, 4 * J);
  Z = std::min<int64_t>(Z, nz);
  d.Z = (int)Z;
  d.G = (int)(ntile * ((nz + Z - 1) / Z));
  if (d.nx_dots)
    k_mpk3d<KIND, J, TXE, TYE, true><<<d.G, TXE * TYE, 0, c.stream>>>(d);
  else
    k_mpk3d<KIND, J, TXE, TYE, false><<<d.G, TXE * TYE, 0, c.stream>>>(d);
}

template <int KIND>
void dispatch_j(Ctx& c, MpkDesc& d) {
  if (d.op.dim == 2) {
    switch (d.J) {
      case 1: launch2d<KIND, 1>(c, d); break;
      case 2: launch2d<KIND, 2>(c, d); break;
      case 3: launch2d<KIND, 3>(c, d); break;
      case 4: launch2d<KIND, 4>(c, d); break;
      case 5: launch2d<KIND, 5>(c, d); break;
      case 6: launch2d<KIND, 6>(c, d); break;
      case 7: launch2d<KIND, 7>(c, d); break;
      default: launch2d<KIND, 8>(c, d); break;
    }
  } else {
    switch (d.J) {
      case 1: launch3d<KIND, 1>(c, d); break;
      case 2: launch3d<KIND, 2>(c, d); break;
      default: launch3d<KIND, 3>(c, d); break;
    }
  }
}

}  // namespace

int mpk_max_depth(const DevOp& op) { return op.kind == kCsr ? 0 : op.dim == 2 ? MPK_MAXJ : 3; }

// Powers of src*scale: out[0] (level 0, may be null) .. out[J].  Products X[x] . level j for
// j >= jdot0 are written at dot0 + x*(J-jdot0+1) + (j-jdot0); returns the partial count G.
int launch_mpk(Ctx& c, const DevOp& op, const double* src, const double* scale, double* const* out, int J,
               int nxd, const double* const* X, int jdot0, double* partials, int dot0, const int* halt,
               const int* cond) {
  require(op.kind != kCsr, "mpk: general CSR operators use repeated applies");
  require(J >= 1 && J <= mpk_max_depth(op), "mpk: depth out of range");
  require(nxd == 0 || (nxd == J + 1 && jdot0 <= 1), "mpk: fused products need J+1 vectors against levels 1..J");
  MpkDesc d;
  std::memset(&d, 0, sizeof d);
  d.op = op;
  d.src = src;
  d.scale = scale;
  for (int j = 0; j <= J; ++j) d.out[j] = out[j];
  d.J = J;
  d.nx_dots = nxd;
  for (int x = 0; x < nxd; ++x) d.X[x] = X[x];
  d.jdot0 = jdot0 < 1 ? 1 : jdot0;
  d.partials = partials;
  d.dot0 = dot0;
  d.halt = halt;
  d.cond = cond;
  // ghost rows of the source from the neighbouring slabs (no-op on one GPU)
  c.halo_exchange(op, src, J);
  int nout = 0;
  for (int j = 0; j <= J; ++j) nout += out[j] != nullptr;
  const double bytes = 8.0 * (double)op.n * (1 + nout + nxd) + (op.kind == kStencilVarK ? 8.0 * op.n : 0.0) +
                       (op.kind == kStencilDia ? 8.0 * (op.dim == 2 ? 5 : 7) * op.n : 0.0);
  Launch lh(c, "mpk", bytes);
  switch (op.kind) {
    case kStencilConst: dispatch_j<kStencilConst>(c, d); break;
    case kStencilVarK: dispatch_j<kStencilVarK>(c, d); break;
    default: dispatch_j<kStencilDia>(c, d); break;
  }
  CK(cudaGetLastError());
  return d.G;
}

}  // namespace skc
