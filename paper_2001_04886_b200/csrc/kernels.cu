// kernels.cu -- streaming kernels of libskrylov_b200 (sm_100a, fp64 CUDA cores).
//
//  * k_apply      : y = A x for the h^2-scaled 5/7-point stencils (constant, variable-k,
//                   per-cell diagonals) and general CSR.  Bit-identical to the reference
//                   spmv (sparse.hpp:135-146): acc = 0, then + v*x per present neighbour
//                   in ascending column order, multiply and add rounded separately.
//  * k_lincomb    : fused block vector update y_o = base_o + sum_j c_jo x_j applied in the
//                   reference's per-element order (axpy / block_axpy_inplace,
//                   kernels.hpp:55-58, block.hpp:109-116) plus inner products of the
//                   results, written as deterministic per-CTA partials.
//  * k_gram       : packed block inner products L^T R (block_gram / block_dot,
//                   block.hpp:70-99) as per-CTA partials.
#include <cstdio>

#include "device_util.cuh"
#include "skc_internal.hpp"

namespace skc {

// ------------------------------------------------------------------ stencil point
__device__ __forceinline__ double face_k(double kp, double kq) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, kp), kq), __dadd_rn(kp, kq));
}

template <int DIM, int KIND>
__device__ __forceinline__ double stencil_point(const DevOp& op, const double* __restrict__ x, int64_t i,
                                                int64_t j, int64_t l) {
  const int64_t nx = op.nx, ny = op.ny;
  const int64_t plane = nx * ny;
  const int64_t p = (DIM == 3 ? l * plane : 0) + j * nx + i;
  bool pres[7];
  int64_t nb[7];
  pres[0] = DIM == 3 && l > 0;
  pres[1] = j > 0;
  pres[2] = i > 0;
  pres[3] = true;
  pres[4] = i + 1 < nx;
  pres[5] = j + 1 < ny;
  pres[6] = DIM == 3 && l + 1 < op.nz;
  nb[0] = p - plane;
  nb[1] = p - nx;
  nb[2] = p - 1;
  nb[3] = p;
  nb[4] = p + 1;
  nb[5] = p + nx;
  nb[6] = p + plane;
  double val[7];
  if (KIND == kStencilConst) {
#pragma unroll
    for (int t = 0; t < 7; ++t) val[t] = op.coef[t];
  } else if (KIND == kStencilDia) {
#pragma unroll
    for (int t = 0; t < 7; ++t) val[t] = (DIM == 2 && (t == 0 || t == 6)) ? 0.0 : op.dia[t * op.n + p];
  } else {  // variable k, faces -z,-y,-x,+x,+y,+z; own k on boundary faces
    const double kp = op.kcell[p];
    double d = 0.0;
    bool first = true;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
      if (t == 3) continue;
      if (DIM == 2 && (t == 0 || t == 6)) continue;
      const double kf = pres[t] ? face_k(kp, op.kcell[nb[t]]) : kp;
      d = first ? kf : __dadd_rn(d, kf);
      first = false;
      val[t] = t < 3 ? __dsub_rn(-kf, op.ch2) : __dadd_rn(-kf, op.ch2);
    }
    val[3] = d;
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    if (DIM == 2 && (t == 0 || t == 6)) continue;
    if (pres[t]) acc = __dadd_rn(acc, __dmul_rn(val[t], x[nb[t]]));
  }
  return acc;
}

template <int DIM, int KIND>
__global__ void __launch_bounds__(256) k_apply(const __grid_constant__ DevOp op, const double* __restrict__ x,
                                               double* __restrict__ y, const int* halt, const int* cond) {
  if (skip_launch(halt, cond)) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  const int64_t l = blockIdx.z;
  if (i >= op.nx) return;
  const int64_t p = (DIM == 3 ? l * op.nx * op.ny : 0) + j * op.nx + i;
  y[p] = stencil_point<DIM, KIND>(op, x, i, j, l);
}

__global__ void __launch_bounds__(256) k_apply_csr(const __grid_constant__ DevOp op, const double* __restrict__ x,
                                                   double* __restrict__ y, const int* halt, const int* cond) {
  if (skip_launch(halt, cond)) return;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= op.n) return;
  double acc = 0.0;
  for (int64_t q = op.rowptr[row]; q < op.rowptr[row + 1]; ++q)
    acc = __dadd_rn(acc, __dmul_rn(op.vals[q], x[op.colidx[q]]));
  y[row] = acc;
}

void launch_apply(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond) {
  const double bytes = 16.0 * op.n + (op.kind == kStencilVarK ? 8.0 * op.n : 0.0) +
                       (op.kind == kStencilDia ? 8.0 * (op.dim == 2 ? 5 : 7) * op.n : 0.0);
  Launch L(c, "apply", bytes);
  if (op.kind == kCsr) {
    const unsigned blocks = (unsigned)((op.n + 255) / 256);
    k_apply_csr<<<blocks, 256, 0, c.stream>>>(op, x, y, halt, cond);
  } else {
    dim3 grid((unsigned)((op.nx + 255) / 256), (unsigned)op.ny, (unsigned)(op.dim == 3 ? op.nz : 1));
    const int key = op.dim * 10 + op.kind;
    switch (key) {
      case 21: k_apply<2, kStencilConst><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      case 22: k_apply<2, kStencilVarK><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      case 23: k_apply<2, kStencilDia><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      case 31: k_apply<3, kStencilConst><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      case 32: k_apply<3, kStencilVarK><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      case 33: k_apply<3, kStencilDia><<<grid, 256, 0, c.stream>>>(op, x, y, halt, cond); break;
      default: fail(SKC_EINVAL, "apply: unsupported operator kind");
    }
  }
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------ block reduction to partials
// acc[k] per thread -> partials[(dot0 + k) * G + blockIdx.x] (fixed order)
template <int K>
__device__ __forceinline__ void block_store_partials(double (&acc)[K], int nk, double* partials, int dot0, int G,
                                                     int gidx, double* red /* >= 8*K */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < nk) {
      const double v = warp_sum(acc[k]);
      if (lane == 0) red[warp * K + k] = v;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w * K + k];
    partials[(int64_t)(dot0 + k) * G + gidx] = s;
  }
}

// ------------------------------------------------------------------ k_lincomb
template <int MAXD>
__global__ void __launch_bounds__(256) k_lincomb(const __grid_constant__ LinDesc d) {
  if (skip_launch(d.halt, d.cond)) return;
  extern __shared__ double smem[];
  double* scoef = smem;                      // ncoef
  double* sv = smem + ((d.ncoef + 1) & ~1);  // (nout + nx) * 256 when MAXD > 0
  for (int t = threadIdx.x; t < d.ncoef; t += blockDim.x) scoef[t] = d.coef[t];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * d.range;
  const int64_t r1 = min(d.n, r0 + d.range);
  double acc[MAXD > 0 ? MAXD : 1];
#pragma unroll
  for (int k = 0; k < (MAXD > 0 ? MAXD : 1); ++k) acc[k] = 0.0;

  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double o[LC_MAXOUT];
#pragma unroll
    for (int q = 0; q < LC_MAXOUT; ++q) {
      if (q < d.nout) {
        double b = d.base[q][i];
        if (d.bscale[q] >= 0) b = dmul(b, scoef[d.bscale[q]]);
        o[q] = b;
      }
    }
    for (int j = 0; j < d.nin; ++j) {
      const double v = d.in[j][i];
      const unsigned m = d.mask[j];
      const double* cj = scoef + d.cbase[j];
#pragma unroll
      for (int q = 0; q < LC_MAXOUT; ++q)
        if ((m >> q) & 1u) o[q] = dadd(o[q], dmul(cj[q], v));
    }
#pragma unroll
    for (int q = 0; q < LC_MAXOUT; ++q)
      if (q < d.nout) d.out[q][i] = o[q];
    if (MAXD > 0) {
      double* col = sv + threadIdx.x;
#pragma unroll
      for (int q = 0; q < LC_MAXOUT; ++q)
        if (q < d.nout) col[q * 256] = o[q];
      for (int x = 0; x < d.nx; ++x) col[(d.nout + x) * 256] = d.xin[x][i];
#pragma unroll
      for (int k = 0; k < (MAXD > 0 ? MAXD : 1); ++k)
        if (k < d.nd) acc[k] = fma(col[d.da[k] * 256], col[d.db[k] * 256], acc[k]);
    }
  }
  if (MAXD > 0) {
    __syncthreads();
    block_store_partials<(MAXD > 0 ? MAXD : 1)>(acc, d.nd, d.partials, d.dot0, d.G, blockIdx.x, sv);
  }
}

void launch_lincomb(Ctx& c, const LinDesc& d, const char* name) {
  require(d.nin <= LC_MAXIN && d.nout <= LC_MAXOUT && d.nx <= LC_MAXX && d.nd <= LC_MAXD, "lincomb: descriptor too large");
  double bytes = 8.0 * (double)d.n * (d.nin + d.nout + d.nx);
  for (int q = 0; q < d.nout; ++q) {  // count each distinct base read once
    bool aliased = false;
    for (int j = 0; j < d.nin; ++j) aliased |= d.in[j] == d.base[q];
    if (!aliased) bytes += 8.0 * (double)d.n;
  }
  Launch L(c, name, bytes);
  const int vals = d.nout + d.nx;
  size_t sm = 8 * (size_t)((d.ncoef + 1) & ~1);
  const int maxd = d.nd == 0 ? 0 : d.nd <= 16 ? 16 : 64;
  if (maxd) sm += 8 * (size_t)std::max(vals * 256, 8 * maxd);
  if (maxd == 0) {
    k_lincomb<0><<<d.G, 256, sm, c.stream>>>(d);
  } else if (maxd == 16) {
    k_lincomb<16><<<d.G, 256, sm, c.stream>>>(d);
  } else {
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(k_lincomb<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      CK(cudaFuncSetAttribute(k_lincomb<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      attr = true;
    }
    k_lincomb<64><<<d.G, 256, sm, c.stream>>>(d);
  }
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------ k_gram
__global__ void __launch_bounds__(256) k_gram(const __grid_constant__ GramDesc d) {
  if (skip_launch(d.halt, d.cond)) return;
  __shared__ double red[8 * GR_LB * GR_MAXR];
  const int64_t r0 = (int64_t)blockIdx.x * d.range;
  const int64_t r1 = min(d.n, r0 + d.range);
  const int l0 = blockIdx.y * GR_LB;
  const int nlb = min(GR_LB, d.nl - l0);
  double acc[GR_LB * GR_MAXR];
#pragma unroll
  for (int k = 0; k < GR_LB * GR_MAXR; ++k) acc[k] = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double rv[GR_MAXR];
#pragma unroll
    for (int r = 0; r < GR_MAXR; ++r) rv[r] = r < d.nr ? d.R[r][i] : 0.0;
#pragma unroll
    for (int lb = 0; lb < GR_LB; ++lb) {
      if (lb < nlb) {
        const double lv = d.L[l0 + lb][i];
#pragma unroll
        for (int r = 0; r < GR_MAXR; ++r)
          if (r < d.nr) acc[lb * GR_MAXR + r] = fma(lv, rv[r], acc[lb * GR_MAXR + r]);
      }
    }
  }
  // reduce: index k = lb*GR_MAXR + r  -> dot (l0+lb)*nr + r
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < GR_LB * GR_MAXR; ++k) {
    const int lb = k / GR_MAXR, r = k % GR_MAXR;
    if (lb < nlb && r < d.nr) {
      const double v = warp_sum(acc[k]);
      if (lane == 0) red[warp * GR_LB * GR_MAXR + k] = v;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < GR_LB * GR_MAXR; k += blockDim.x) {
    const int lb = k / GR_MAXR, r = k % GR_MAXR;
    if (lb < nlb && r < d.nr) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w * GR_LB * GR_MAXR + k];
      d.partials[(int64_t)(d.dot0 + (l0 + lb) * d.nr + r) * d.G + blockIdx.x] = s;
    }
  }
}

void launch_gram(Ctx& c, const GramDesc& d, const char* name) {
  require(d.nl >= 1 && d.nl <= GR_MAXL && d.nr >= 1 && d.nr <= GR_MAXR, "gram: descriptor out of range");
  double bytes = 8.0 * (double)d.n * d.nr;
  for (int l = 0; l < d.nl; ++l) {
    bool dup = false;
    for (int r = 0; r < d.nr; ++r) dup |= d.L[l] == d.R[r];
    if (!dup) bytes += 8.0 * (double)d.n;
  }
  Launch L(c, name, bytes);
  dim3 grid(d.G, (d.nl + GR_LB - 1) / GR_LB);
  k_gram<<<grid, 256, 0, c.stream>>>(d);
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------ misc
__global__ void k_fill(double* p, double v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void launch_fill(Ctx& c, double* p, double v, int64_t n) {
  ++c.launches;
  k_fill<<<std::min<int64_t>(1184, (n + 255) / 256 + 1), 256, 0, c.stream>>>(p, v, n);
  CK(cudaGetLastError());
}

}  // namespace skc
