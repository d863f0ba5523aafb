// mpk.cu -- matrix-powers kernel: [v, A v, ..., A^J v] of v = src * scale for the 5-point
// (2D) and 7-point (3D) stencils in one pass over src, with a width-J ghost zone.
//
// Replaces krylov_block (block.hpp:59-67) / krylov_pair (sstep.hpp:71-81): each power is
// bit-identical to J successive reference spmv calls (sparse.hpp:135-146) because every
// stencil point is evaluated in the reference's ascending-column order with separately
// rounded multiplies and adds; out-of-domain neighbours enter as exact zeros, which leaves
// the sum's bits unchanged (adding +-0.0 to a sum that starts at +0.0).
//
// 2D: a warp owns an output strip of W columns x R rows and streams it in y (no block-level
// synchronisation: x-neighbours by warp shuffles, y-neighbours in registers).  Level j at
// step t produces row t-j.  3D: a CTA owns an (x,y) tile extended by J on each side and
// streams it in z; each level's newest plane is shared through double-buffered shared memory
// with one __syncthreads per plane step.
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

// Source rows are staged into shared-memory rings by per-thread cp.async copies (each thread
// copies its own column(s); one commit group per row step), PF rows ahead of the row being
// consumed.  The ring has PF+1 slots: a step refills the slot consumed one step earlier.  With
// DOTS the X rows of the row the last level completes ride in the same groups.
//
// Stencil value at a point: S, W, C, E, N (2D) or -z,-y,-x,C,+x,+y,+z (3D) in ascending column
// order with separately rounded multiplies and adds; absent neighbours are exact zeros.

// ------------------------------------------------------------------ 2D
// Warp strips: a warp owns W = 64 - 2J output columns (two adjacent columns per lane, J ghost
// columns each side) of R rows and streams them in y with no block-level synchronisation:
// level j keeps its last three rows per column in registers (the y-neighbours), and the
// x-neighbours of a lane's column pair are the adjacent lanes' columns, read with warp
// shuffles.  Lane-edge columns see a neighbour from the wrong end of the warp; they are ghost
// columns, and level j is valid on columns [j, 64-j) of the strip, so the J levels leave the
// W middle columns exact.  Source rows (and, with DOTS, the X rows of the row the last level
// completes) arrive PF rows ahead through per-lane cp.async rings in shared memory.
constexpr int MW_WARPS = 4;           // independent strips per CTA
constexpr int MW_PF = 4, MW_NS = 5;   // prefetch distance, ring slots (PF + 1)

template <int J, bool DOTS>
constexpr size_t mpk2w_smem() {
  return sizeof(double) * MW_WARPS * 64 * MW_NS * (1 + (DOTS ? (size_t)J + 1 : 0));
}

template <int KIND>
__device__ __forceinline__ double point2d(const DevOp& op, int64_t r, int64_t rg, int64_t rows_g, int c, int nx,
                                          double ys, double xw, double cc, double xe, double yn) {
  double cS, cW, cC, cE, cN;
  const bool hasS = rg > 0, hasN = rg + 1 < rows_g, hasW = c > 0, hasE = c + 1 < nx;
  if (KIND == kStencilConst) {
    cS = op.coef[1], cW = op.coef[2], cC = op.coef[3], cE = op.coef[4], cN = op.coef[5];
  } else {
    bool pres[7];
    int64_t nb[7];
    const int64_t p = r * nx + c;
    pres[0] = pres[6] = false;
    pres[1] = hasS;
    pres[2] = hasW;
    pres[3] = true;
    pres[4] = hasE;
    pres[5] = hasN;
    nb[0] = nb[6] = nb[3] = p;
    nb[1] = p - nx;
    nb[2] = p - 1;
    nb[4] = p + 1;
    nb[5] = p + nx;
    double val[7];
    coefs<2, KIND>(op, p, pres, nb, val);
    cS = val[1], cW = val[2], cC = val[3], cE = val[4], cN = val[5];
  }
  double a = 0.0;
  a = __dadd_rn(a, __dmul_rn(cS, hasS ? ys : 0.0));
  a = __dadd_rn(a, __dmul_rn(cW, hasW ? xw : 0.0));
  a = __dadd_rn(a, __dmul_rn(cC, cc));
  a = __dadd_rn(a, __dmul_rn(cE, hasE ? xe : 0.0));
  a = __dadd_rn(a, __dmul_rn(cN, hasN ? yn : 0.0));
  return a;
}

template <int KIND, int J, bool DOTS>
__global__ void __launch_bounds__(MW_WARPS * 32) k_mpk2w(const __grid_constant__ MpkDesc d) {
  SKC_PDL_ENTRY();
  static_assert(!DOTS || J <= 3, "fused products read level values from the 3-row windows");
  if (skip_launch(d.halt, d.cond)) return;
  constexpr int PF = MW_PF, NS = MW_NS, NX = J + 1;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* ring = dsm + (size_t)wid * NS * 64;                        // [NS][64] per warp
  double* xring = dsm + (size_t)MW_WARPS * NS * 64 + (size_t)wid * NX * NS * 64;  // [NX][NS][64]
  const int nx = (int)d.op.nx, ny = (int)d.op.ny;
  const int task = blockIdx.x * MW_WARPS + wid;
  const bool active = task < d.tiles_x * d.tiles_y;  // warp-uniform
  const int tx = active ? task % d.tiles_x : 0, ty = active ? task / d.tiles_x : 0;
  const int y0 = ty * d.R, y1 = min(ny, y0 + d.R);
  const int ca = tx * d.W - J + 2 * lane, cb = ca + 1;  // this lane's columns
  const bool inA = ca >= 0 && ca < nx, inB = cb >= 0 && cb < nx;
  const bool outA = 2 * lane >= J && 2 * lane < J + d.W && inA;
  const bool outB = 2 * lane + 1 >= J && 2 * lane + 1 < J + d.W && inB;
  const double scale = d.scale ? *d.scale : 1.0;
  double wa[J + 1][3], wb[J + 1][3];  // per level: rows (r-1, r, r+1), columns a and b
#pragma unroll
  for (int j = 0; j <= J; ++j) wa[j][0] = wa[j][1] = wa[j][2] = wb[j][0] = wb[j][1] = wb[j][2] = 0.0;
  constexpr int NACC = DOTS ? NX * J : 1;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  // slab geometry: local row t is global row row0 + t; rows just outside the slab come from
  // the halo buffers (filled by the exchange), rows outside the grid are Dirichlet zeros
  const int row0 = (int)d.op.row0, rows_g = (int)d.op.rows_global;
  const int H = (int)d.op.halo_rows;
  const int tb = y0 - J, te = y1 + J;
  // lane constants: neighbour presence of the two columns, the outputs, the constant stencil
  const bool hWa = ca > 0, hEa = cb < nx, hWb = ca >= 0, hEb = cb + 1 < nx;
  double* outs[J + 1];
#pragma unroll
  for (int j = 0; j <= J; ++j) outs[j] = d.out[j];
  double cS = 0.0, cW = 0.0, cC = 0.0, cE = 0.0, cN = 0.0;
  if (KIND == kStencilConst) cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
  auto issue = [&](int t) {
    const int slot = (t - tb) % NS;
    const int tg = row0 + t;
    const bool rowok = active && tg >= 0 && tg < rows_g && t < te;
    const double* rowp = d.src;
    if (rowok)
      rowp = t < 0 ? d.op.hlo + (int64_t)(t + H) * nx
                   : (t >= ny ? d.op.hhi + (int64_t)(t - ny) * nx : d.src + (int64_t)t * nx);
    double* rs = ring + slot * 64 + 2 * lane;
    cp_async8(rs, rowok && inA ? rowp + ca : d.src, rowok && inA);
    cp_async8(rs + 1, rowok && inB ? rowp + cb : d.src, rowok && inB);
    if (DOTS) {
      const int r = t - J;
      const bool rok = active && r >= y0 && r < y1;
#pragma unroll
      for (int x = 0; x < NX; ++x) {
        const double* xr = d.X[x] + (int64_t)r * nx;
        double* xs = xring + (x * NS + slot) * 64 + 2 * lane;
        cp_async8(xs, rok && outA ? xr + ca : d.src, rok && outA);
        cp_async8(xs + 1, rok && outB ? xr + cb : d.src, rok && outB);
      }
    }
    cp_async_commit();
  };
  if (active) {
#pragma unroll 1
    for (int k = 0; k < PF; ++k) issue(tb + k);
#pragma unroll 1
    for (int t = tb; t < te; ++t) {
      const int slot = (t - tb) % NS;
      cp_async_wait<PF - 1>();
      const bool rowin = row0 + t >= 0 && row0 + t < rows_g;
      {
        const double sa = ring[slot * 64 + 2 * lane], sb = ring[slot * 64 + 2 * lane + 1];
        const double va = inA && rowin ? (d.scale ? __dmul_rn(sa, scale) : sa) : 0.0;
        const double vb = inB && rowin ? (d.scale ? __dmul_rn(sb, scale) : sb) : 0.0;
        wa[0][0] = wa[0][1], wa[0][1] = wa[0][2], wa[0][2] = va;
        wb[0][0] = wb[0][1], wb[0][1] = wb[0][2], wb[0][2] = vb;
        if (outs[0] && t >= y0 && t < y1) {
          double* o = outs[0] + (int64_t)t * nx;
          if (outA) o[ca] = va;
          if (outB) o[cb] = vb;
        }
      }
#pragma unroll
      for (int j = 1; j <= J; ++j) {
        const int r = t - j;  // row level j computes
        const int rg = row0 + r;
        // x-neighbours of level j-1 at row r
        const double ma = wa[j - 1][1], mb = wb[j - 1][1];
        const double wA = __shfl_up_sync(FULL, mb, 1);    // column ca-1 (lane-1's b)
        const double eB = __shfl_down_sync(FULL, ma, 1);  // column cb+1 (lane+1's a)
        // level j is needed (and its inputs valid) only within J-j rows of the warp's rows
        const bool rv = rg >= 0 && rg < rows_g && r >= y0 - (J - j) && r < y1 + (J - j);  // warp-uniform
        double va, vb;
        if (KIND == kStencilConst) {
          // S, W, C, E, N (ascending column), separately rounded; absent neighbours are zeros
          const bool hS = rg > 0, hN = rg + 1 < rows_g;
          double a = 0.0, b = 0.0;
          a = __dadd_rn(a, __dmul_rn(cS, hS ? wa[j - 1][0] : 0.0));
          b = __dadd_rn(b, __dmul_rn(cS, hS ? wb[j - 1][0] : 0.0));
          a = __dadd_rn(a, __dmul_rn(cW, hWa ? wA : 0.0));
          b = __dadd_rn(b, __dmul_rn(cW, hWb ? ma : 0.0));
          a = __dadd_rn(a, __dmul_rn(cC, ma));
          b = __dadd_rn(b, __dmul_rn(cC, mb));
          a = __dadd_rn(a, __dmul_rn(cE, hEa ? mb : 0.0));
          b = __dadd_rn(b, __dmul_rn(cE, hEb ? eB : 0.0));
          a = __dadd_rn(a, __dmul_rn(cN, hN ? wa[j - 1][2] : 0.0));
          b = __dadd_rn(b, __dmul_rn(cN, hN ? wb[j - 1][2] : 0.0));
          va = rv && inA ? a : 0.0;
          vb = rv && inB ? b : 0.0;
        } else {
          va = 0.0, vb = 0.0;
          if (rv) {
            if (inA) va = point2d<KIND>(d.op, r, rg, rows_g, ca, nx, wa[j - 1][0], wA, ma, mb, wa[j - 1][2]);
            if (inB) vb = point2d<KIND>(d.op, r, rg, rows_g, cb, nx, wb[j - 1][0], ma, mb, eB, wb[j - 1][2]);
          }
        }
        wa[j][0] = wa[j][1], wa[j][1] = wa[j][2], wa[j][2] = va;
        wb[j][0] = wb[j][1], wb[j][1] = wb[j][2], wb[j][2] = vb;
        if (outs[j] && r >= y0 && r < y1) {
          double* o = outs[j] + (int64_t)r * nx;
          if (outA) o[ca] = va;
          if (outB) o[cb] = vb;
        }
      }
      // products of row t-J, complete at every level: level j's value sits J-j rows back
      if (DOTS) {
        const int r = t - J;
        if (r >= y0 && r < y1) {
#pragma unroll
          for (int x = 0; x < NX; ++x) {
            const double* xs = xring + (x * NS + slot) * 64 + 2 * lane;
            const double xa = xs[0], xb = xs[1];  // zero-filled outside the output columns
#pragma unroll
            for (int j = 1; j <= J; ++j) {
              acc[x * J + (j - 1)] = fma(xa, wa[j][2 - (J - j)], acc[x * J + (j - 1)]);
              acc[x * J + (j - 1)] = fma(xb, wb[j][2 - (J - j)], acc[x * J + (j - 1)]);
            }
          }
        }
      }
      issue(t + PF);  // refills the slot consumed at step t-1 (its reads retired in order)
    }
  }
  if (DOTS) {
    // fixed-order CTA reduction: product (x, level j) -> dot0 + x*J + (j-1)
    __shared__ double red[MW_WARPS][NACC];
    warp_sums(acc, red[wid]);
    __syncthreads();
    for (int e = threadIdx.x; e < NACC; e += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < MW_WARPS; ++w) s += red[w][e];
      d.partials[(int64_t)(d.dot0 + e) * kPartialPitch + blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------ 3D
// tile: TXE x TYE threads (extended by J each side), streamed over d.Z planes
constexpr int PF3 = 4;

template <int J, int NT, bool DOTS>
constexpr size_t mpk3d_smem() {
  return sizeof(double) * NT * ((size_t)2 * J + (PF3 + 1) * (DOTS ? (size_t)J + 2 : 1));
}

template <int KIND, int J, int TXE, int TYE, bool DOTS>
__global__ void __launch_bounds__(TXE* TYE) k_mpk3d(const __grid_constant__ MpkDesc d) {
  SKC_PDL_ENTRY();
  static_assert(!DOTS || J <= 3, "fused products read level values from the 3-row windows");
  if (skip_launch(d.halt, d.cond)) return;
  constexpr int NT = TXE * TYE, PF = PF3, NS = PF3 + 1, NX = J + 1;
  extern __shared__ __align__(16) double dsm[];
  double* plane = dsm;                 // [J][2][TYE][TXE]
  double* ring = plane + 2 * J * NT;   // [NS][NT]
  double* xring = ring + NS * NT;      // [NX][NS][NT]
  const int tid = threadIdx.x;
  const int lx = tid % TXE, ly = tid / TXE;
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
  constexpr int NACC = DOTS ? NX * J : 1;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;

  // z-slab geometry (see the 2D kernel): plane t is global plane row0 + t
  const int64_t row0 = d.op.row0, rows_g = d.op.rows_global;
  const int64_t H = d.op.halo_rows;
  const int64_t xy = y * nx + x;
  const int64_t tb = z0 - J, te = z1 + J;
  auto issue = [&](int64_t t) {
    const int slot = (int)((t - tb) % NS);
    const int64_t tg = row0 + t;
    const bool ok = in && tg >= 0 && tg < rows_g && t < te;
    const double* pp = d.src;
    if (ok) pp = (t < 0 ? d.op.hlo + (t + H) * pl : (t >= nz ? d.op.hhi + (t - nz) * pl : d.src + t * pl)) + xy;
    cp_async8(ring + slot * NT + tid, pp, ok);
    if (DOTS) {
      const int64_t r = t - J;
      const bool okx = outp && r >= z0 && r < z1;
#pragma unroll
      for (int q = 0; q < NX; ++q) cp_async8(xring + (q * NS + slot) * NT + tid, okx ? d.X[q] + r * pl + xy : d.src, okx);
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int k = 0; k < PF; ++k) issue(tb + k);
#pragma unroll 1
  for (int64_t t = tb; t < te; ++t) {
    const int par = (int)(t & 1);
    const int slot = (int)((t - tb) % NS);
    cp_async_wait<PF - 1>();
    const double s0 = ring[slot * NT + tid];
    double v0 = 0.0;
    if (in && row0 + t >= 0 && row0 + t < rows_g) v0 = d.scale ? __dmul_rn(s0, scale) : s0;
    win[0][0] = win[0][1];
    win[0][1] = win[0][2];
    win[0][2] = v0;
    plane[par * NT + tid] = v0;
    if (d.out[0] && outp && t >= z0 && t < z1) d.out[0][t * pl + xy] = v0;
#pragma unroll
    for (int j = 1; j <= J; ++j) {
      const int64_t r = t - j;  // plane computed by level j
      const int64_t rg = row0 + r;
      double v = 0.0;
      if (in && rg >= 0 && rg < rows_g && r >= z0 - (J - j) && r < z1 + (J - j)) {
        const double* P = plane + ((j - 1) * 2 + (par ^ 1)) * NT;
        const double ys = ly > 0 ? P[tid - TXE] : 0.0;
        const double xw = lx > 0 ? P[tid - 1] : 0.0;
        const double xe = lx + 1 < TXE ? P[tid + 1] : 0.0;
        const double yn = ly + 1 < TYE ? P[tid + TXE] : 0.0;
        bool pres[7];
        int64_t nb[7];
        const int64_t p = r * pl + xy;
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
      if (j < J) plane[(j * 2 + par) * NT + tid] = v;
      if (d.out[j] && outp && r >= z0 && r < z1) d.out[j][r * pl + xy] = v;
    }
    if (DOTS) {
      const int64_t r = t - J;
      if (outp && r >= z0 && r < z1) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
          const double xv = xring[(q * NS + slot) * NT + tid];
#pragma unroll
          for (int j = 1; j <= J; ++j) acc[q * J + (j - 1)] = fma(xv, win[j][2 - (J - j)], acc[q * J + (j - 1)]);
        }
      }
    }
    issue(t + PF);
    __syncthreads();
  }
  if (DOTS) {
    constexpr int NW = NT / 32;
    __shared__ double red[NW][NACC];
    const int warp = tid >> 5;
    warp_sums(acc, red[warp]);
    __syncthreads();
    for (int e = tid; e < NACC; e += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += red[w][e];
      d.partials[(int64_t)(d.dot0 + e) * kPartialPitch + blockIdx.x] = s;
    }
  }
}

// Small 2D grids (single GPU, no fused products): one CTA per 32 x 32 tile extended by J on each
// side, all J levels computed in shared memory with one __syncthreads per level.  The row-
// streaming strip kernel needs ~R + 2J dependent row steps per strip, which dominates when
// the whole grid is only a few dozen strips (C1: 128 x 128); here a launch is one load round
// trip plus J on-chip levels.  Level j is exact on [j, 32 - j) of the tile, so the output
// (the inner 32 - 2J square) is bit-identical to J successive spmv calls, as in the other
// kernels.
constexpr int T2 = 32;
template <int KIND, int J>
__global__ void __launch_bounds__(T2* T2) k_mpk2t(const __grid_constant__ MpkDesc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.halt, d.cond)) return;
  __shared__ double lev[2][T2 * T2];
  const int tid = threadIdx.x;
  const int lx = tid % T2, ly = tid / T2;
  const int tx = blockIdx.x % d.tiles_x, ty = blockIdx.x / d.tiles_x;
  const int64_t nx = d.op.nx, ny = d.op.ny;
  const int64_t x = (int64_t)tx * d.W - J + lx, y = (int64_t)ty * d.R - J + ly;
  const bool in = x >= 0 && x < nx && y >= 0 && y < ny;
  const bool outp = lx >= J && lx < T2 - J && ly >= J && ly < T2 - J && x < nx && y < ny;
  const int64_t p = y * nx + x;
  double v = 0.0;
  if (in) v = d.scale ? __dmul_rn(d.src[p], *d.scale) : d.src[p];
  lev[0][tid] = v;
  if (d.out[0] && outp) d.out[0][p] = v;
  bool pres[7];
  int64_t nb[7];
  pres[0] = pres[6] = false;
  pres[1] = y > 0;
  pres[2] = x > 0;
  pres[3] = true;
  pres[4] = x + 1 < nx;
  pres[5] = y + 1 < ny;
  nb[0] = nb[6] = p;
  nb[1] = p - nx;
  nb[2] = p - 1;
  nb[3] = p;
  nb[4] = p + 1;
  nb[5] = p + nx;
  double val[7];
  if (in) coefs<2, KIND>(d.op, p, pres, nb, val);
#pragma unroll
  for (int j = 1; j <= J; ++j) {
    __syncthreads();
    const double* P = lev[(j - 1) & 1];
    double a = 0.0;
    if (in && lx >= j && lx < T2 - j && ly >= j && ly < T2 - j) {
      a = __dadd_rn(a, __dmul_rn(val[1], pres[1] ? P[tid - T2] : 0.0));
      a = __dadd_rn(a, __dmul_rn(val[2], pres[2] ? P[tid - 1] : 0.0));
      a = __dadd_rn(a, __dmul_rn(val[3], P[tid]));
      a = __dadd_rn(a, __dmul_rn(val[4], pres[4] ? P[tid + 1] : 0.0));
      a = __dadd_rn(a, __dmul_rn(val[5], pres[5] ? P[tid + T2] : 0.0));
    }
    lev[j & 1][tid] = a;
    if (d.out[j] && outp) d.out[j][p] = a;
  }
}


template <int KIND, int J, bool DOTS>
void run2d(Ctx& c, const MpkDesc& d) {
  constexpr size_t smem = mpk2w_smem<J, DOTS>();
  ensure_smem(k_mpk2w<KIND, J, DOTS>, smem);
  launch_k(c, k_mpk2w<KIND, J, DOTS>, d.G, MW_WARPS * 32, smem, d);
}

// resident CTAs per SM of the strip kernel, at most 4 (the geometry the fused products' partial
// layout was sized for); cached per device (the attribute call precedes the query)
template <int KIND, int J>
int mpk2w_resident(Ctx& c, bool dots) {
  static int cache[2][64] = {};
  int& slot = cache[dots ? 1 : 0][c.device & 63];
  if (slot) return slot;
  int per_sm = 0;
  if constexpr (J <= 3) {
    if (dots) {
      ensure_smem(k_mpk2w<KIND, J, true>, mpk2w_smem<J, true>());
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mpk2w<KIND, J, true>, MW_WARPS * 32,
                                                       mpk2w_smem<J, true>()));
      return slot = std::min(4, std::max(1, per_sm));
    }
  }
  ensure_smem(k_mpk2w<KIND, J, false>, mpk2w_smem<J, false>());
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mpk2w<KIND, J, false>, MW_WARPS * 32,
                                                   mpk2w_smem<J, false>()));
  return slot = std::min(4, std::max(1, per_sm));
}

template <int KIND, int J>
void launch2d(Ctx& c, MpkDesc& d) {
  const int64_t nx = d.op.nx, ny = d.op.ny;
  if (J <= 8 && !d.nx_dots && d.op.halo_rows == 0 && d.op.rows_global == ny) {
    const int64_t tw = T2 - 2 * J;
    const int64_t ntile = ((nx + tw - 1) / tw) * ((ny + tw - 1) / tw);
    if (ntile <= 2LL * c.sm_count) {  // the strip kernel would leave most SMs idle
      d.W = d.R = (int)tw;
      d.tiles_x = (int)((nx + tw - 1) / tw);
      d.tiles_y = (int)((ny + tw - 1) / tw);
      d.G = (int)ntile;
      launch_k(c, k_mpk2t<KIND, J>, d.G, T2 * T2, 0, d);
      return;
    }
  }
  d.W = 64 - 2 * J;
  d.tiles_x = (int)((nx + d.W - 1) / d.W);
  // rows per warp strip: the strips fill whole waves of resident CTAs (a grid a little over one
  // wave runs two: C4's 656 CTAs on 592 slots streamed at 3.5 TB/s), at least 3J rows per strip
  // to bound the ghost-row overhead
  bool dots = false;
  if constexpr (J <= 3) dots = d.nx_dots != 0;
  const int64_t slots = (int64_t)mpk2w_resident<KIND, J>(c, dots) * c.sm_count * MW_WARPS;  // strips per wave
  const int64_t ty_max = std::max<int64_t>(1, ny / (3 * J));
  int64_t ty = std::max<int64_t>(1, slots / d.tiles_x);
  if (ty > ty_max) {  // many short strips: whole waves as far as the 3J rows allow
    const int64_t waves = (d.tiles_x * ty_max + slots - 1) / slots;
    ty = std::max<int64_t>(1, std::min(ty_max, waves * slots / d.tiles_x));
  }
  const int64_t R = std::min<int64_t>(ny, (ny + ty - 1) / ty);
  d.R = (int)R;
  d.tiles_y = (int)((ny + R - 1) / R);
  d.G = (d.tiles_x * d.tiles_y + MW_WARPS - 1) / MW_WARPS;
  if constexpr (J <= 3) {
    if (d.nx_dots) return run2d<KIND, J, true>(c, d);
  }
  run2d<KIND, J, false>(c, d);
}

template <int KIND, int J, bool DOTS>
void run3d(Ctx& c, const MpkDesc& d) {
  constexpr int TXE = 32, TYE = 16;
  constexpr size_t smem = mpk3d_smem<J, TXE * TYE, DOTS>();
  ensure_smem(k_mpk3d<KIND, J, TXE, TYE, DOTS>, smem);
  launch_k(c, k_mpk3d<KIND, J, TXE, TYE, DOTS>, d.G, TXE * TYE, smem, d);
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
    run3d<KIND, J, true>(c, d);
  else
    run3d<KIND, J, false>(c, d);
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

int mpk_max_depth(const DevOp& op) { return op.kind == kCsr || op.kind == kIlu0 ? 0 : op.dim == 2 ? MPK_MAXJ : 3; }
// on one GPU the constant 3D stencil takes the one-sweep 2.5D kernel (mpk3.cu, depth <= 4); the
// other 3D operators the single-level applies (the ghost-zone tile sweep of k_mpk3d loses to
// them there); slabs need k_mpk3d for the halos
int powers_depth(const Ctx& c, const DevOp& op) {
  if (op.dim == 3 && c.world() == 1) return op.kind == kStencilConst && c.mpk3 ? 4 : 0;
  return mpk_max_depth(op);
}

// Powers of src*scale: out[0] (level 0, may be null) .. out[J].  Products X[x] . level j for
// j >= jdot0 are written at dot0 + x*(J-jdot0+1) + (j-jdot0); returns the partial count G.
int launch_mpk(Ctx& c, const DevOp& op, const double* src, const double* scale, double* const* out, int J,
               int nxd, const double* const* X, int jdot0, double* partials, int dot0, const int* halt,
               const int* cond, const char* name) {
  require(op.kind != kCsr, "mpk: general CSR operators use repeated applies");
  if (nxd == 0 && c.world() == 1 && c.mpk3 && launch_mpk3(c, op, src, scale, out, J, halt, cond, name)) return 0;
  require(J >= 1 && J <= mpk_max_depth(op), "mpk: depth out of range");
  require(nxd == 0 || (nxd == J + 1 && jdot0 <= 1 && J <= kMpkMaxDotDepth),
          "mpk: fused products need J+1 vectors against levels 1..J (J <= 3)");
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
  Launch lh(c, name, bytes);
  switch (op.kind) {
    case kStencilConst: dispatch_j<kStencilConst>(c, d); break;
    case kStencilVarK: dispatch_j<kStencilVarK>(c, d); break;
    default: dispatch_j<kStencilDia>(c, d); break;
  }
  CK(cudaGetLastError());
  return d.G;
}

}  // namespace skc
