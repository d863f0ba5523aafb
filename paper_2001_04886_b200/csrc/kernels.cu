// kernels.cu -- streaming kernels of libskrylov_b200 (sm_100a, fp64 CUDA cores).
//
//  * k_apply      : y = A x for the h^2-scaled 5/7-point stencils (constant, variable-k,
//                   per-cell diagonals) and general CSR.  Bit-identical to the reference
//                   spmv (sparse.hpp:135-146): acc = 0, then + v*x per present neighbour
//                   in ascending column order, multiply and add rounded separately.
// The streaming update / inner-product kernels live in stream.cu.
#include <cstdio>

#include "device_util.cuh"
#include "skc_internal.hpp"
#include "stencil.cuh"

namespace skc {

template <int DIM, int KIND>
__global__ void __launch_bounds__(256) k_apply(const __grid_constant__ DevOp op, const double* __restrict__ x,
                                               double* __restrict__ y, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
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
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= op.n) return;
  double acc = 0.0;
  for (int64_t q = op.rowptr[row]; q < op.rowptr[row + 1]; ++q)
    acc = __dadd_rn(acc, __dmul_rn(op.vals[q], x[op.colidx[q]]));
  y[row] = acc;
}

void launch_apply(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond) {
  if (op.kind != kCsr && c.world() > 1) {  // slabs: depth-1 matrix-powers sweep (halo exchange)
    double* outs[2] = {nullptr, y};
    launch_mpk(c, op, x, nullptr, outs, 1, 0, nullptr, 1, nullptr, 0, halt, cond);
    return;
  }
  const double bytes = 16.0 * op.n + (op.kind == kStencilVarK ? 8.0 * op.n : 0.0) +
                       (op.kind == kStencilDia ? 8.0 * (op.dim == 2 ? 5 : 7) * op.n : 0.0);
  Launch L(c, "apply", bytes);
  if (op.kind == kCsr) {
    const unsigned blocks = (unsigned)((op.n + 255) / 256);
    launch_k(c, k_apply_csr, blocks, 256, 0, op, x, y, halt, cond);
  } else {
    dim3 grid((unsigned)((op.nx + 255) / 256), (unsigned)op.ny, (unsigned)(op.dim == 3 ? op.nz : 1));
    const int key = op.dim * 10 + op.kind;
    switch (key) {
      case 21: launch_k(c, k_apply<2, kStencilConst>, grid, 256, 0, op, x, y, halt, cond); break;
      case 22: launch_k(c, k_apply<2, kStencilVarK>, grid, 256, 0, op, x, y, halt, cond); break;
      case 23: launch_k(c, k_apply<2, kStencilDia>, grid, 256, 0, op, x, y, halt, cond); break;
      case 31: launch_k(c, k_apply<3, kStencilConst>, grid, 256, 0, op, x, y, halt, cond); break;
      case 32: launch_k(c, k_apply<3, kStencilVarK>, grid, 256, 0, op, x, y, halt, cond); break;
      case 33: launch_k(c, k_apply<3, kStencilDia>, grid, 256, 0, op, x, y, halt, cond); break;
      default: fail(SKC_EINVAL, "apply: unsupported operator kind");
    }
  }
  CK(cudaGetLastError());
}

// ------------------------------------------------------------------ misc
__global__ void k_fill(double* p, double v, int64_t n) {
  SKC_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

void launch_fill(Ctx& c, double* p, double v, int64_t n) {
  ++c.launches;
  launch_k(c, k_fill, std::min<int64_t>(1184, (n + 255) / 256 + 1), 256, 0, p, v, n);
  CK(cudaGetLastError());
}

}  // namespace skc
