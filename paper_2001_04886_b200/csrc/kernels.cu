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

// 3D variable-k stencil, z-marching, every face coefficient computed once: a 32 x 8 thread tile
// of (x, y) columns walks KZ planes.  The harmonic-mean face coefficient 2 kp kq / (kp + kq)
// (one fp64 division) is symmetric in its bits (2 kp is exact, the product and the sum
// commute), so a thread computes only its +x, +y and +z faces and takes -x from the lane to
// its left (lane 0 of a row is a halo column: the tiles overlap by one column in x), -y from
// the thread row below through shared memory (row 0 of the tile recomputes it: a warp-uniform
// branch) and -z from its own previous plane -- 3 + 1/8 + 1/16 divisions per point instead of
// 6.  The x values of a column stay in registers across planes as in k_apply3z.  Same
// arithmetic order as stencil_point (faces -z,-y,-x,+x,+y,+z; own k on boundary faces).
constexpr int AV_TX = 32, AV_TY = 8, AV_KZ = 16;
__global__ void __launch_bounds__(AV_TX* AV_TY) k_apply3z_vark(const __grid_constant__ DevOp op,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  __shared__ double sfn[2][AV_TY][AV_TX];  // the +y faces of a plane (double-buffered)
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % AV_TX, ty = threadIdx.x / AV_TX;
  const int i = blockIdx.x * (AV_TX - 1) + tx - 1;  // (lane 0: the halo column to the left)
  const int j = blockIdx.y * AV_TY + ty;
  const bool in = i >= 0 && i < nx && j < ny;
  const bool outp = in && tx > 0;
  const int l0 = blockIdx.z * AV_KZ, l1 = min(nz, l0 + AV_KZ);
  const int64_t plane = (int64_t)nx * ny;
  const double ch2 = op.ch2;
  const bool hW = in && i > 0, hE = in && i + 1 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* xc_ = x + c;
  const double* kc_ = op.kcell + c;
  double xm = in && l0 > 0 ? __ldg(xc_ + (int64_t)(l0 - 1) * plane) : 0.0;
  double xc = in ? __ldg(xc_ + (int64_t)l0 * plane) : 0.0;
  double kc = in ? __ldg(kc_ + (int64_t)l0 * plane) : 1.0;
  double fzm = kc;  // the -z face (own k at the domain boundary)
  if (l0 > 0) {     // (block-uniform)
    const double km = in ? __ldg(kc_ + (int64_t)(l0 - 1) * plane) : 1.0;
    fzm = face_k(kc, km);
  }
  for (int l = l0; l < l1; ++l) {
    const int64_t o = (int64_t)l * plane;
    const bool hZ = l + 1 < nz;
    const double xp = in && hZ ? __ldg(xc_ + o + plane) : 0.0;
    const double kp = in && hZ ? __ldg(kc_ + o + plane) : 1.0;
    const double kE = hE ? __ldg(kc_ + o + 1) : 1.0, kN = hN ? __ldg(kc_ + o + nx) : 1.0;
    const double vs = hS ? __ldg(xc_ + o - nx) : 0.0, vw = hW ? __ldg(xc_ + o - 1) : 0.0;
    const double ve = hE ? __ldg(xc_ + o + 1) : 0.0, vn = hN ? __ldg(xc_ + o + nx) : 0.0;
    const double fE = hE ? face_k(kc, kE) : kc;
    const double fN = hN ? face_k(kc, kN) : kc;
    const double fZ = hZ ? face_k(kc, kp) : kc;
    sfn[l & 1][ty][tx] = fN;
    double fW = __shfl_up_sync(0xffffffffu, fE, 1);
    if (!hW) fW = kc;
    __syncthreads();
    double fS;
    if (ty > 0) {
      fS = hS ? sfn[l & 1][ty - 1][tx] : kc;
    } else {  // (warp-uniform: the tile's first row)
      const double kS = hS ? __ldg(kc_ + o - nx) : 1.0;
      fS = hS ? face_k(kc, kS) : kc;
    }
    if (outp) {
      double dsum = fzm;
      dsum = __dadd_rn(dsum, fS);
      dsum = __dadd_rn(dsum, fW);
      dsum = __dadd_rn(dsum, fE);
      dsum = __dadd_rn(dsum, fN);
      dsum = __dadd_rn(dsum, fZ);
      double a = 0.0;
      if (l > 0) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fzm, ch2), xm));
      if (hS) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fS, ch2), vs));
      if (hW) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fW, ch2), vw));
      a = __dadd_rn(a, __dmul_rn(dsum, xc));
      if (hE) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fE, ch2), ve));
      if (hN) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fN, ch2), vn));
      if (hZ) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fZ, ch2), xp));
      y[o + c] = a;
    }
    xm = xc;
    xc = xp;
    kc = kp;
    fzm = fZ;
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
      case 32: {
        const dim3 gz((unsigned)((op.nx + AV_TX - 2) / (AV_TX - 1)), (unsigned)((op.ny + AV_TY - 1) / AV_TY),
                      (unsigned)((op.nz + AV_KZ - 1) / AV_KZ));
        launch_k(c, k_apply3z_vark, gz, AV_TX * AV_TY, 0, op, x, y, halt, cond);
        break;
      }
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
