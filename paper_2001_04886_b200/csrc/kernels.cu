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

// 3D constant stencil, z-marching: a 32 x 8 thread tile of (x, y) columns walks KZ planes; the
// -z / centre / +z values of a column stay in registers (one new plane load per point), the
// x / y neighbours come through L1.  Same arithmetic order as stencil_point.
constexpr int AZ_TX = 32, AZ_TY = 8, AZ_KZ = 16;
__global__ void __launch_bounds__(AZ_TX* AZ_TY) k_apply3z(const __grid_constant__ DevOp op,
                                                         const double* __restrict__ x, double* __restrict__ y,
                                                         const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int i = blockIdx.x * AZ_TX + threadIdx.x % AZ_TX;
  const int j = blockIdx.y * AZ_TY + threadIdx.x / AZ_TX;
  if (i >= nx || j >= ny) return;
  const int l0 = blockIdx.z * AZ_KZ, l1 = min(nz, l0 + AZ_KZ);
  const int64_t plane = (int64_t)nx * ny;
  const double c0 = op.coef[0], c1 = op.coef[1], c2 = op.coef[2], c3 = op.coef[3], c4 = op.coef[4],
               c5 = op.coef[5], c6 = op.coef[6];
  const bool hW = i > 0, hE = i + 1 < nx, hS = j > 0, hN = j + 1 < ny;
  const double* col = x + (int64_t)j * nx + i;
  double zm = l0 > 0 ? __ldg(col + (int64_t)(l0 - 1) * plane) : 0.0;
  double zc = __ldg(col + (int64_t)l0 * plane);
  for (int l = l0; l < l1; ++l) {
    const double* pc = col + (int64_t)l * plane;
    const double zp = l + 1 < nz ? __ldg(pc + plane) : 0.0;
    const double vs = hS ? __ldg(pc - nx) : 0.0, vw = hW ? __ldg(pc - 1) : 0.0;
    const double ve = hE ? __ldg(pc + 1) : 0.0, vn = hN ? __ldg(pc + nx) : 0.0;
    double a = 0.0;
    if (l > 0) a = __dadd_rn(a, __dmul_rn(c0, zm));
    if (hS) a = __dadd_rn(a, __dmul_rn(c1, vs));
    if (hW) a = __dadd_rn(a, __dmul_rn(c2, vw));
    a = __dadd_rn(a, __dmul_rn(c3, zc));
    if (hE) a = __dadd_rn(a, __dmul_rn(c4, ve));
    if (hN) a = __dadd_rn(a, __dmul_rn(c5, vn));
    if (l + 1 < nz) a = __dadd_rn(a, __dmul_rn(c6, zp));
    y[(int64_t)l * plane + (int64_t)j * nx + i] = a;
    zm = zc;
    zc = zp;
  }
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
  if (op.kind == kIlu0) {  // y = A (LU)^{-1} x (right_preconditioned, ilu0.hpp:138-146)
    double* tmp = (double*)c.workspace("ilu_apply_tmp", sizeof(double) * (size_t)op.n);
    launch_ilu0_solve(c, *op.ilu, x, tmp, halt, cond);
    launch_apply(c, op.ilu->base.d, tmp, y, halt, cond);
    return;
  }
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
      case 31: {
        const dim3 gz((unsigned)((op.nx + AZ_TX - 1) / AZ_TX), (unsigned)((op.ny + AZ_TY - 1) / AZ_TY),
                      (unsigned)((op.nz + AZ_KZ - 1) / AZ_KZ));
        launch_k(c, k_apply3z, gz, AZ_TX * AZ_TY, 0, op, x, y, halt, cond);
        break;
      }
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
