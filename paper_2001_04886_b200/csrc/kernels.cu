// kernels.cu -- streaming kernels of libskrylov_b200 (sm_100a, fp64 CUDA cores).
//
//  * k_apply      : y = A x for the h^2-scaled 5/7-point stencils (constant, variable-k,
//                   per-cell diagonals) and general CSR.  Bit-identical to the reference
//                   spmv (sparse.hpp:135-146): acc = 0, then + v*x per present neighbour
//                   in ascending column order, multiply and add rounded separately.
// The streaming update / inner-product kernels live in stream.cu.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

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

// 3D variable-k stencil from stored face coefficients.  The harmonic means of a cell's +x, +y
// and +z faces (own k on the domain boundary) are computed once when the operator is built
// (k_faces3: the same face_k bits the on-the-fly kernels produce, and symmetric, so a cell's -x
// face is its left neighbour's +x face); the apply is then a division-free stream of x, the
// three face arrays and y (40 bytes per point instead of 24 plus 3.2 divisions).  z-marching
// 32 x 8 tiles: the -z face and the x column stay in registers across planes, the W / E
// values and the -x face come from the adjacent lanes (the warp's edge lanes load them), the
// y neighbours through L1.  Same arithmetic order as stencil_point.
constexpr int AF_TX = 32, AF_TY = 8, AF_KZ = 16;
__global__ void __launch_bounds__(256) k_faces3(const __grid_constant__ DevOp op, double* __restrict__ f) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= op.n) return;
  const int64_t plane = op.nx * op.ny;
  const int64_t i = p % op.nx, j = (p / op.nx) % op.ny, l = p / plane;
  const double kp = op.kcell[p];
  f[p] = i + 1 < op.nx ? face_k(kp, op.kcell[p + 1]) : kp;
  f[op.n + p] = j + 1 < op.ny ? face_k(kp, op.kcell[p + op.nx]) : kp;
  f[2 * op.n + p] = l + 1 < op.nz ? face_k(kp, op.kcell[p + plane]) : kp;
}

void launch_faces3(Ctx& c, const DevOp& op, double* faces) {
  k_faces3<<<(unsigned)((op.n + 255) / 256), 256, 0, c.stream>>>(op, faces);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c.stream));
}

__global__ void __launch_bounds__(AF_TX* AF_TY) k_apply3z_face(const __grid_constant__ DevOp op,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int lane = threadIdx.x % AF_TX;
  const int i = blockIdx.x * AF_TX + lane;
  const int j = blockIdx.y * AF_TY + threadIdx.x / AF_TX;
  if (j >= ny) return;  // (warp-uniform; lanes past nx stay for the shuffles)
  const bool in = i < nx;
  const int l0 = blockIdx.z * AF_KZ, l1 = min(nz, l0 + AF_KZ);
  const int64_t plane = (int64_t)nx * ny;
  const double ch2 = op.ch2;
  const bool hW = in && i > 0, hE = in && i + 1 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool ldW = hW && lane == 0, ldE = hE && lane == AF_TX - 1;
  const bool needk = in && (i == 0 || j == 0);
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* xc_ = x + c;
  const double* fx = op.faces + c;
  const double* fy = fx + op.n;
  const double* fz = fy + op.n;
  const double* kc_ = op.kcell + c;
  double xm = in && l0 > 0 ? __ldg(xc_ + (int64_t)(l0 - 1) * plane) : 0.0;
  double xc = in ? __ldg(xc_ + (int64_t)l0 * plane) : 0.0;
  // the -z face: the cell below's +z face, own k on the domain boundary
  double fzm = !in ? 0.0 : l0 > 0 ? __ldg(fz + (int64_t)(l0 - 1) * plane) : __ldg(kc_);
  for (int l = l0; l < l1; ++l) {
    const int64_t o = (int64_t)l * plane;
    const bool hZ = l + 1 < nz;
    const double xp = in && hZ ? __ldg(xc_ + o + plane) : 0.0;
    const double fE = in ? __ldg(fx + o) : 0.0, fN = in ? __ldg(fy + o) : 0.0, fZ = in ? __ldg(fz + o) : 0.0;
    const double kc = needk ? __ldg(kc_ + o) : 0.0;
    const double vs = hS ? __ldg(xc_ + o - nx) : 0.0, vn = hN ? __ldg(xc_ + o + nx) : 0.0;
    double fW = __shfl_up_sync(0xffffffffu, fE, 1);
    double vw = __shfl_up_sync(0xffffffffu, xc, 1);
    double ve = __shfl_down_sync(0xffffffffu, xc, 1);
    if (ldW) {
      fW = __ldg(fx + o - 1);
      vw = __ldg(xc_ + o - 1);
    }
    if (ldE) ve = __ldg(xc_ + o + 1);
    if (!hW) fW = kc;
    const double fS = hS ? __ldg(fy + o - nx) : kc;
    if (in) {
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
    fzm = fZ;
  }
}

// ---- 3D applies through a shared-memory plane ring.  The z-marching kernels above keep one
// plane of loads in flight per thread (the loop stalls on them before the next plane's are
// issued), which bounds them at ~3.5-3.9 TB/s whatever the tile shape or the bytes per point
// (measured: constant stencil 16 B/point 3.8 TB/s, stored faces 40 B/point 3.5 TB/s).  Here every
// thread copies its point of plane l+1+D (and the tile's halo) with cp.async into a ring of
// D+2 plane slots while plane l is computed from shared memory: D planes of every CTA are in
// flight with no register cost.  One CTA barrier per plane; the column's x(l-1) and the -z face
// stay in registers.  Same arithmetic order as stencil_point.
constexpr int AR_TX = 32, AR_TY = 8;
constexpr int AR_W = AR_TX + 2, AR_H = AR_TY + 2;

template <int D>
__global__ void __launch_bounds__(AR_TX* AR_TY) k_apply3r(const __grid_constant__ DevOp op,
                                                         const double* __restrict__ x, double* __restrict__ y,
                                                         int kz, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  constexpr int NS = D + 2;
  __shared__ double ring[NS][AR_H][AR_W];
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % AR_TX, ty = threadIdx.x / AR_TX;
  const int i = blockIdx.x * AR_TX + tx;
  const int j = blockIdx.y * AR_TY + ty;
  const bool in = i < nx && j < ny;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double c0 = op.coef[0], c1 = op.coef[1], c2 = op.coef[2], c3 = op.coef[3], c4 = op.coef[4],
               c5 = op.coef[5], c6 = op.coef[6];
  const bool hW = in && i > 0, hE = in && i + 1 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool cW = hW && tx == 0, cE = hE && tx == AR_TX - 1, cS = hS && ty == 0, cN = hN && ty == AR_TY - 1;
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* col = x + c;
  // plane q -> slot q mod NS (planes l0 .. min(l1, nz-1); one commit group per call, empty past the end)
  auto issue = [&](int q, int slot) {
    if (q <= l1 && q < nz) {
      const double* src = col + (int64_t)q * plane;
      double(*pl)[AR_W] = ring[slot];
      cp_async8(&pl[ty + 1][tx + 1], src, in);
      if (cW) cp_async8(&pl[ty + 1][0], src - 1, true);
      if (cE) cp_async8(&pl[ty + 1][AR_W - 1], src + 1, true);
      if (cS) cp_async8(&pl[0][tx + 1], src - nx, true);
      if (cN) cp_async8(&pl[AR_H - 1][tx + 1], src + nx, true);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q <= D; ++q) issue(l0 + q, q);
  double xm = in && l0 > 0 ? __ldg(col + (int64_t)(l0 - 1) * plane) : 0.0;
  int sc = 0;       // slot of plane l
  int sn = D + 1;   // slot of plane l + 1 + D (= the slot of plane l - 1)
  for (int l = l0; l < l1; ++l) {
    cp_async_wait<D - 1>();  // planes l and l + 1 have landed (this thread's copies)
    __syncthreads();         // ... everyone's; and plane l - 1's slot is no longer read
    issue(l + 1 + D, sn);
    const int s1 = sc + 1 == NS ? 0 : sc + 1;
    if (in) {
      const double(*pl)[AR_W] = ring[sc];
      const double zc = pl[ty + 1][tx + 1];
      double a = 0.0;
      if (l > 0) a = __dadd_rn(a, __dmul_rn(c0, xm));
      if (hS) a = __dadd_rn(a, __dmul_rn(c1, pl[ty][tx + 1]));
      if (hW) a = __dadd_rn(a, __dmul_rn(c2, pl[ty + 1][tx]));
      a = __dadd_rn(a, __dmul_rn(c3, zc));
      if (hE) a = __dadd_rn(a, __dmul_rn(c4, pl[ty + 1][tx + 2]));
      if (hN) a = __dadd_rn(a, __dmul_rn(c5, pl[ty + 2][tx + 1]));
      if (l + 1 < nz) a = __dadd_rn(a, __dmul_rn(c6, ring[s1][ty + 1][tx + 1]));
      y[(int64_t)l * plane + c] = a;
      xm = zc;
    }
    sc = s1;
    sn = sn + 1 == NS ? 0 : sn + 1;
  }
  cp_async_wait<0>();
}

// Column pairs: a thread owns two adjacent points of a row (16-byte copies, loads and stores; nx
// even), so a tile row is 2 x 256 / TY points wide -- 512 B to 2 KB of contiguous memory per row
// instead of 256 B, which is what DRAM wants -- and there is half the copy / load / store
// instruction count per point.  Row layout in a slot: [pad, W, TX points, E, pad].
template <int D, int TY>
__global__ void __launch_bounds__(256) k_apply3r2(const __grid_constant__ DevOp op, const double* __restrict__ x,
                                                  double* __restrict__ y, int kz, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  constexpr int NS = D + 2, TXP = 256 / TY, TX = 2 * TXP, W = TX + 4, H = TY + 2;
  extern __shared__ __align__(16) double ring2[];  // [NS][H][W]
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % TXP, ty = threadIdx.x / TXP;
  const int i = blockIdx.x * TX + 2 * tx;  // the pair i, i + 1 (both inside: nx is even)
  const int j = blockIdx.y * TY + ty;
  const bool in = i < nx && j < ny;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double c0 = op.coef[0], c1 = op.coef[1], c2 = op.coef[2], c3 = op.coef[3], c4 = op.coef[4],
               c5 = op.coef[5], c6 = op.coef[6];
  const bool hW = in && i > 0, hE = in && i + 2 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool cW = hW && tx == 0, cE = hE && tx == TXP - 1, cS = hS && ty == 0, cN = hN && ty == TY - 1;
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* col = x + c;
  const int oc = (ty + 1) * W + 2 + 2 * tx;  // the pair's offset inside a slot
  auto issue = [&](int q, int slot) {
    if (q <= l1 && q < nz) {
      const double* src = col + (int64_t)q * plane;
      double* sl = ring2 + slot * (H * W);
      cp_async16(sl + oc, src, in);
      if (cW) cp_async8(sl + oc - 1, src - 1, true);
      if (cE) cp_async8(sl + oc + 2, src + 2, true);
      if (cS) cp_async16(sl + oc - W, src - nx, true);
      if (cN) cp_async16(sl + oc + W, src + nx, true);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q <= D; ++q) issue(l0 + q, q);
  double2 xm = make_double2(0.0, 0.0);
  if (in && l0 > 0) xm = *reinterpret_cast<const double2*>(col + (int64_t)(l0 - 1) * plane);
  int sc = 0, sn = D + 1;
  for (int l = l0; l < l1; ++l) {
    cp_async_wait<D - 1>();
    __syncthreads();
    issue(l + 1 + D, sn);
    const int s1 = sc + 1 == NS ? 0 : sc + 1;
    if (in) {
      const double* sl = ring2 + sc * (H * W) + oc;
      const double2 C = *reinterpret_cast<const double2*>(sl);
      double a0 = 0.0, a1 = 0.0;
      if (l > 0) {
        a0 = __dadd_rn(a0, __dmul_rn(c0, xm.x));
        a1 = __dadd_rn(a1, __dmul_rn(c0, xm.y));
      }
      if (hS) {
        const double2 S = *reinterpret_cast<const double2*>(sl - W);
        a0 = __dadd_rn(a0, __dmul_rn(c1, S.x));
        a1 = __dadd_rn(a1, __dmul_rn(c1, S.y));
      }
      if (hW) a0 = __dadd_rn(a0, __dmul_rn(c2, sl[-1]));
      a1 = __dadd_rn(a1, __dmul_rn(c2, C.x));
      a0 = __dadd_rn(a0, __dmul_rn(c3, C.x));
      a1 = __dadd_rn(a1, __dmul_rn(c3, C.y));
      a0 = __dadd_rn(a0, __dmul_rn(c4, C.y));
      if (hE) a1 = __dadd_rn(a1, __dmul_rn(c4, sl[2]));
      if (hN) {
        const double2 N = *reinterpret_cast<const double2*>(sl + W);
        a0 = __dadd_rn(a0, __dmul_rn(c5, N.x));
        a1 = __dadd_rn(a1, __dmul_rn(c5, N.y));
      }
      if (l + 1 < nz) {
        const double2 Z = *reinterpret_cast<const double2*>(ring2 + s1 * (H * W) + oc);
        a0 = __dadd_rn(a0, __dmul_rn(c6, Z.x));
        a1 = __dadd_rn(a1, __dmul_rn(c6, Z.y));
      }
      *reinterpret_cast<double2*>(y + (int64_t)l * plane + c) = make_double2(a0, a1);
      xm = C;
    }
    sc = s1;
    sn = sn + 1 == NS ? 0 : sn + 1;
  }
  cp_async_wait<0>();
}

template <int D, int TY>
static void launch_apply3r2(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond);

// The same ring fed by the TMA engine: x is described to the hardware as a 3D tensor
// (nx, ny, nz) and one thread asks for a whole plane tile with its halo -- the box
// [i0 - 2, i0 + TX + 2) x [j0 - 1, j0 + TY + 1) of plane q -- with one
// cp.async.bulk.tensor.3d (SASS UTMALDG); coordinates outside the grid are zero-filled by the
// unit, and each slot's mbarrier counts the box's bytes in.  The other 255 threads issue no
// copies, compute no halo addresses and wait on no copy groups: the ring can run NS - 1 planes
// ahead for one instruction per plane.  (Two columns of left halo instead of one keep the
// pairs 16-byte aligned in the slot; a slot is padded to a multiple of 128 bytes.)
constexpr int AT_TXP = 64, AT_TX = 2 * AT_TXP, AT_W = AT_TX + 4;
// R = rows per thread (rows ty, ty + 4, ...): a tile is 4 R rows, a slot (4 R + 2) x AT_W doubles
// padded to a multiple of 128 bytes
template <int R>
struct AtGeo {
  static constexpr int TY = 4 * R, H = TY + 2, BOX = AT_W * H * 8, SLOT = ((BOX + 127) / 128) * 16;
};
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
template <int NS, int R, bool DN = false, bool EF = false>
__global__ void __launch_bounds__(256, R == 1 ? 8 : R == 2 ? 5 : 3) k_apply3t(const __grid_constant__ CUtensorMap tm,
                                                 const __grid_constant__ DevOp op, const double* __restrict__ x,
                                                 double* __restrict__ y, int kz, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  using G = AtGeo<R>;
  extern __shared__ __align__(128) double ringt[];  // [NS][SLOT], then NS mbarriers
  uint64_t* full = reinterpret_cast<uint64_t*>(ringt + NS * G::SLOT);
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % AT_TXP, ty = threadIdx.x / AT_TXP;
  const int i0 = blockIdx.x * AT_TX, j0 = blockIdx.y * G::TY;
  const int i = i0 + 2 * tx;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double c0 = op.coef[0], c1 = op.coef[1], c2 = op.coef[2], c3 = op.coef[3], c4 = op.coef[4],
               c5 = op.coef[5], c6 = op.coef[6];
  const bool hW = i > 0, hE = i + 2 < nx;
  const int oc = (ty + 1) * AT_W + 2 + 2 * tx;  // the pair's offset inside a slot (row ty)
  // the planes are walked upwards (plane(p) = l0 + p, then plane l1 for its z neighbour) or, DN,
  // downwards (plane(p) = l1 - 1 - p, then plane l0 - 1): chained applies alternate so that one
  // starts on the planes its predecessor wrote last, still in L2
  const int cnt = (l1 - l0) + ((DN ? l0 > 0 : l1 < nz) ? 1 : 0);  // planes this CTA reads
  uint64_t pol = 0;
  if (EF) pol = policy_evict_first();
  const bool lead = threadIdx.x == 0;
  if (lead) {
#pragma unroll
    for (int st = 0; st < NS; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int p) {  // plane l0 + p into slot p % NS (the leader)
    if (p < cnt) {
      const int st = p % NS;
      mbar_arrive_expect_tx(&full[st], G::BOX);
      if (EF)
        tma_load_3d_hint(ringt + st * G::SLOT, &tm, i0 - 2, j0 - 1, DN ? l1 - 1 - p : l0 + p, &full[st], pol);
      else
        tma_load_3d(ringt + st * G::SLOT, &tm, i0 - 2, j0 - 1, DN ? l1 - 1 - p : l0 + p, &full[st]);
    }
  };
  if (lead) {
#pragma unroll
    for (int p = 0; p < NS - 1; ++p) issue(p);
  }
  bool in[R];
  double2 xm[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int j = j0 + ty + 4 * r;
    in[r] = i < nx && j < ny;
    xm[r] = make_double2(0.0, 0.0);
    if (in[r] && (DN ? l1 < nz : l0 > 0))
      xm[r] = *reinterpret_cast<const double2*>(x + (int64_t)j * nx + i + (int64_t)(DN ? l1 : l0 - 1) * plane);
  }
  double* yp = y + (int64_t)(j0 + ty) * nx + i + (int64_t)(DN ? l1 - 1 : l0) * plane;
  mbar_wait(&full[0], 0);
  int sc = 0, s1 = 1 % NS;
  uint32_t par1 = 0;  // parity of the phase plane p + 1 completes in its slot
  for (int p = 0; p < l1 - l0; ++p) {
    const int l = DN ? l1 - 1 - p : l0 + p;
    __syncthreads();  // everyone is done with plane p - 1: its slot takes plane p + NS - 1
    if (lead) issue(p + NS - 1);
    const bool hZ = l + 1 < nz, hB = l > 0;
    if (DN ? hB : hZ) mbar_wait(&full[s1], par1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (in[r]) {
        const int j = j0 + ty + 4 * r;
        const double* sl = ringt + sc * G::SLOT + oc + 4 * r * AT_W;
        const double2 C = *reinterpret_cast<const double2*>(sl);
        double a0 = 0.0, a1 = 0.0;
        if (hB) {
          const double2 B = DN ? *reinterpret_cast<const double2*>(ringt + s1 * G::SLOT + oc + 4 * r * AT_W) : xm[r];
          a0 = __dadd_rn(a0, __dmul_rn(c0, B.x));
          a1 = __dadd_rn(a1, __dmul_rn(c0, B.y));
        }
        if (j > 0) {
          const double2 S = *reinterpret_cast<const double2*>(sl - AT_W);
          a0 = __dadd_rn(a0, __dmul_rn(c1, S.x));
          a1 = __dadd_rn(a1, __dmul_rn(c1, S.y));
        }
        if (hW) a0 = __dadd_rn(a0, __dmul_rn(c2, sl[-1]));
        a1 = __dadd_rn(a1, __dmul_rn(c2, C.x));
        a0 = __dadd_rn(a0, __dmul_rn(c3, C.x));
        a1 = __dadd_rn(a1, __dmul_rn(c3, C.y));
        a0 = __dadd_rn(a0, __dmul_rn(c4, C.y));
        if (hE) a1 = __dadd_rn(a1, __dmul_rn(c4, sl[2]));
        if (j + 1 < ny) {
          const double2 N = *reinterpret_cast<const double2*>(sl + AT_W);
          a0 = __dadd_rn(a0, __dmul_rn(c5, N.x));
          a1 = __dadd_rn(a1, __dmul_rn(c5, N.y));
        }
        if (hZ) {
          const double2 Z = DN ? xm[r] : *reinterpret_cast<const double2*>(ringt + s1 * G::SLOT + oc + 4 * r * AT_W);
          a0 = __dadd_rn(a0, __dmul_rn(c6, Z.x));
          a1 = __dadd_rn(a1, __dmul_rn(c6, Z.y));
        }
        *reinterpret_cast<double2*>(yp + (int64_t)(4 * r) * nx) = make_double2(a0, a1);
        xm[r] = C;
      }
    }
    yp += DN ? -plane : plane;
    sc = s1;
    s1 = s1 + 1 == NS ? 0 : s1 + 1;
    if (s1 == 0) par1 ^= 1u;
  }
}

// stored-face variable-k form of the same ring: a slot holds the x tile with its halo, the +x
// faces with the column to the left, the +y faces with the row below, and the +z faces
constexpr int AF2_FX = AR_W * AR_H;                 // offsets inside a slot (doubles)
constexpr int AF2_FY = AF2_FX + AR_TY * (AR_TX + 1);
constexpr int AF2_FZ = AF2_FY + (AR_TY + 1) * AR_TX;
constexpr int AF2_SLOT = AF2_FZ + AR_TY * AR_TX;

template <int D>
__global__ void __launch_bounds__(AR_TX* AR_TY) k_apply3r_face(const __grid_constant__ DevOp op,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              int kz, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  constexpr int NS = D + 2;
  extern __shared__ __align__(16) double fring[];  // [NS][AF2_SLOT]
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % AR_TX, ty = threadIdx.x / AR_TX;
  const int i = blockIdx.x * AR_TX + tx;
  const int j = blockIdx.y * AR_TY + ty;
  const bool in = i < nx && j < ny;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double ch2 = op.ch2;
  const bool hW = in && i > 0, hE = in && i + 1 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool cW = hW && tx == 0, cE = hE && tx == AR_TX - 1, cS = hS && ty == 0, cN = hN && ty == AR_TY - 1;
  const bool needk = in && (i == 0 || j == 0);
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* col = x + c;
  const double* fx = op.faces + c;
  const double* fy = fx + op.n;
  const double* fz = fy + op.n;
  const double* kc_ = op.kcell + c;
  const int ox = (ty + 1) * AR_W + tx + 1;            // own x
  const int ofx = AF2_FX + ty * (AR_TX + 1) + tx + 1;  // own +x face (the -x face at ofx - 1)
  const int ofy = AF2_FY + (ty + 1) * AR_TX + tx;      // own +y face (the -y face at ofy - AR_TX)
  const int ofz = AF2_FZ + ty * AR_TX + tx;
  auto issue = [&](int q, int slot) {
    if (q <= l1 && q < nz) {
      const int64_t o = (int64_t)q * plane;
      double* sl = fring + slot * AF2_SLOT;
      cp_async8(sl + ox, col + o, in);
      if (cW) cp_async8(sl + ox - 1, col + o - 1, true);
      if (cE) cp_async8(sl + ox + 1, col + o + 1, true);
      if (cS) cp_async8(sl + ox - AR_W, col + o - nx, true);
      if (cN) cp_async8(sl + ox + AR_W, col + o + nx, true);
      if (q < l1) {  // (the plane past the chunk only lends its x)
        cp_async8(sl + ofx, fx + o, in);
        cp_async8(sl + ofy, fy + o, in);
        cp_async8(sl + ofz, fz + o, in);
        if (cW) cp_async8(sl + ofx - 1, fx + o - 1, true);
        if (cS) cp_async8(sl + ofy - AR_TX, fy + o - nx, true);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q <= D; ++q) issue(l0 + q, q);
  double xm = in && l0 > 0 ? __ldg(col + (int64_t)(l0 - 1) * plane) : 0.0;
  // the -z face: the cell below's +z face, own k on the domain boundary
  double fzm = !in ? 0.0 : l0 > 0 ? __ldg(fz + (int64_t)(l0 - 1) * plane) : __ldg(kc_);
  int sc = 0, sn = D + 1;
  for (int l = l0; l < l1; ++l) {
    cp_async_wait<D - 1>();
    __syncthreads();
    issue(l + 1 + D, sn);
    const int s1 = sc + 1 == NS ? 0 : sc + 1;
    if (in) {
      const double* sl = fring + sc * AF2_SLOT;
      const bool hZ = l + 1 < nz;
      const double kc = needk ? __ldg(kc_ + (int64_t)l * plane) : 0.0;
      const double xc = sl[ox];
      const double fE = sl[ofx], fN = sl[ofy], fZ = sl[ofz];
      const double fW = hW ? sl[ofx - 1] : kc;
      const double fS = hS ? sl[ofy - AR_TX] : kc;
      double dsum = fzm;
      dsum = __dadd_rn(dsum, fS);
      dsum = __dadd_rn(dsum, fW);
      dsum = __dadd_rn(dsum, fE);
      dsum = __dadd_rn(dsum, fN);
      dsum = __dadd_rn(dsum, fZ);
      double a = 0.0;
      if (l > 0) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fzm, ch2), xm));
      if (hS) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fS, ch2), sl[ox - AR_W]));
      if (hW) a = __dadd_rn(a, __dmul_rn(__dsub_rn(-fW, ch2), sl[ox - 1]));
      a = __dadd_rn(a, __dmul_rn(dsum, xc));
      if (hE) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fE, ch2), sl[ox + 1]));
      if (hN) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fN, ch2), sl[ox + AR_W]));
      if (hZ) a = __dadd_rn(a, __dmul_rn(__dadd_rn(-fZ, ch2), fring[s1 * AF2_SLOT + ox]));
      y[(int64_t)l * plane + c] = a;
      xm = xc;
      fzm = fZ;
    }
    sc = s1;
    sn = sn + 1 == NS ? 0 : sn + 1;
  }
  cp_async_wait<0>();
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

// column-pair form of the stored-face ring (nx even): 8 rows of 64 points per tile, 16-byte copies
namespace fp {
constexpr int TY = 8, TXP = 32, TX = 2 * TXP;
constexpr int XW = TX + 4, XH = TY + 2;       // x tile rows: [pad, W, TX points, E, pad]
constexpr int FXW = TX + 2;                   // +x faces: [pad, the column to the left, TX faces]
constexpr int OFX = XW * XH;
constexpr int OFY = OFX + TY * FXW;           // +y faces: the row below, then TY rows of TX
constexpr int OFZ = OFY + (TY + 1) * TX;
constexpr int SLOT = OFZ + TY * TX;
}  // namespace fp

template <int D>
__global__ void __launch_bounds__(256) k_apply3r2_face(const __grid_constant__ DevOp op, const double* __restrict__ x,
                                                       double* __restrict__ y, int kz, const int* halt,
                                                       const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  using namespace fp;
  constexpr int NS = D + 2;
  extern __shared__ __align__(16) double fring2[];  // [NS][SLOT]
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % TXP, ty = threadIdx.x / TXP;
  const int i = blockIdx.x * TX + 2 * tx;
  const int j = blockIdx.y * TY + ty;
  const bool in = i < nx && j < ny;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double ch2 = op.ch2;
  const bool hW = in && i > 0, hE = in && i + 2 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool cW = hW && tx == 0, cE = hE && tx == TXP - 1, cS = hS && ty == 0, cN = hN && ty == TY - 1;
  const bool needk = in && (i == 0 || j == 0);
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* col = x + c;
  const double* fx = op.faces + c;
  const double* fy = fx + op.n;
  const double* fz = fy + op.n;
  const double* kc_ = op.kcell + c;
  const int ox = (ty + 1) * XW + 2 + 2 * tx;
  const int ofx = OFX + ty * FXW + 2 + 2 * tx;
  const int ofy = OFY + (ty + 1) * TX + 2 * tx;
  const int ofz = OFZ + ty * TX + 2 * tx;
  auto issue = [&](int q, int slot) {
    if (q <= l1 && q < nz) {
      const int64_t o = (int64_t)q * plane;
      double* sl = fring2 + slot * SLOT;
      cp_async16(sl + ox, col + o, in);
      if (cW) cp_async8(sl + ox - 1, col + o - 1, true);
      if (cE) cp_async8(sl + ox + 2, col + o + 2, true);
      if (cS) cp_async16(sl + ox - XW, col + o - nx, true);
      if (cN) cp_async16(sl + ox + XW, col + o + nx, true);
      if (q < l1) {
        cp_async16(sl + ofx, fx + o, in);
        cp_async16(sl + ofy, fy + o, in);
        cp_async16(sl + ofz, fz + o, in);
        if (cW) cp_async8(sl + ofx - 1, fx + o - 1, true);
        if (cS) cp_async16(sl + ofy - TX, fy + o - nx, true);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q <= D; ++q) issue(l0 + q, q);
  double2 xm = make_double2(0.0, 0.0), fzm = xm;
  if (in) {
    if (l0 > 0) {
      xm = *reinterpret_cast<const double2*>(col + (int64_t)(l0 - 1) * plane);
      fzm = *reinterpret_cast<const double2*>(fz + (int64_t)(l0 - 1) * plane);
    } else {
      fzm = *reinterpret_cast<const double2*>(kc_);  // own k on the domain boundary
    }
  }
  int sc = 0, sn = D + 1;
  for (int l = l0; l < l1; ++l) {
    cp_async_wait<D - 1>();
    __syncthreads();
    issue(l + 1 + D, sn);
    const int s1 = sc + 1 == NS ? 0 : sc + 1;
    if (in) {
      const double* sl = fring2 + sc * SLOT;
      const bool hZ = l + 1 < nz;
      double2 kc = make_double2(0.0, 0.0);
      if (needk) kc = *reinterpret_cast<const double2*>(kc_ + (int64_t)l * plane);
      const double2 C = *reinterpret_cast<const double2*>(sl + ox);
      const double2 fE = *reinterpret_cast<const double2*>(sl + ofx);
      const double2 fN = *reinterpret_cast<const double2*>(sl + ofy);
      const double2 fZ = *reinterpret_cast<const double2*>(sl + ofz);
      const double fW0 = hW ? sl[ofx - 1] : kc.x;
      const double fW1 = fE.x;  // (the pair's shared face)
      double2 fS = kc, S = make_double2(0.0, 0.0), N = S, Z = S;
      if (hS) {
        fS = *reinterpret_cast<const double2*>(sl + ofy - TX);
        S = *reinterpret_cast<const double2*>(sl + ox - XW);
      }
      if (hN) N = *reinterpret_cast<const double2*>(sl + ox + XW);
      if (hZ) Z = *reinterpret_cast<const double2*>(fring2 + s1 * SLOT + ox);
      double d0 = fzm.x, d1 = fzm.y;
      d0 = __dadd_rn(d0, fS.x);
      d1 = __dadd_rn(d1, fS.y);
      d0 = __dadd_rn(d0, fW0);
      d1 = __dadd_rn(d1, fW1);
      d0 = __dadd_rn(d0, fE.x);
      d1 = __dadd_rn(d1, fE.y);
      d0 = __dadd_rn(d0, fN.x);
      d1 = __dadd_rn(d1, fN.y);
      d0 = __dadd_rn(d0, fZ.x);
      d1 = __dadd_rn(d1, fZ.y);
      double a0 = 0.0, a1 = 0.0;
      if (l > 0) {
        a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fzm.x, ch2), xm.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fzm.y, ch2), xm.y));
      }
      if (hS) {
        a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fS.x, ch2), S.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fS.y, ch2), S.y));
      }
      if (hW) a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fW0, ch2), sl[ox - 1]));
      a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fW1, ch2), C.x));
      a0 = __dadd_rn(a0, __dmul_rn(d0, C.x));
      a1 = __dadd_rn(a1, __dmul_rn(d1, C.y));
      a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fE.x, ch2), C.y));
      if (hE) a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fE.y, ch2), sl[ox + 2]));
      if (hN) {
        a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fN.x, ch2), N.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fN.y, ch2), N.y));
      }
      if (hZ) {
        a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fZ.x, ch2), Z.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fZ.y, ch2), Z.y));
      }
      *reinterpret_cast<double2*>(y + (int64_t)l * plane + c) = make_double2(a0, a1);
      xm = C;
      fzm = fZ;
    }
    sc = s1;
    sn = sn + 1 == NS ? 0 : sn + 1;
  }
  cp_async_wait<0>();
}

// The stored-face ring fed by the TMA engine (see k_apply3t): four boxes per plane -- the x tile
// with its halo, the +x faces with the column to the left, the +y faces with the row below, the
// +z faces -- land in one slot on one mbarrier.  The slot layout is fp's with every box on a
// 128-byte boundary.
namespace fpt {
constexpr int TY = 8, TXP = 32, TX = 2 * TXP;
constexpr int XW = TX + 4, XH = TY + 2, FXW = TX + 2;
constexpr int BX = XW * XH * 8, BFX = FXW * TY * 8, BFY = TX * (TY + 1) * 8, BFZ = TX * TY * 8;  // box bytes
constexpr int pad16(int bytes) { return ((bytes + 127) / 128) * 16; }
constexpr int OFX = pad16(BX);
constexpr int OFY = OFX + pad16(BFX);
constexpr int OFZ = OFY + pad16(BFY);
constexpr int SLOT = OFZ + pad16(BFZ);
}  // namespace fpt
template <int NS>
__global__ void __launch_bounds__(256) k_apply3t_face(const __grid_constant__ CUtensorMap tmx,
                                                      const __grid_constant__ CUtensorMap tmfx,
                                                      const __grid_constant__ CUtensorMap tmfy,
                                                      const __grid_constant__ CUtensorMap tmfz,
                                                      const __grid_constant__ DevOp op, const double* __restrict__ x,
                                                       double* __restrict__ y, int kz, const int* halt,
                                                       const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  using namespace fpt;
  extern __shared__ __align__(128) double fring2[];  // [NS][SLOT], then NS mbarriers
  uint64_t* full = reinterpret_cast<uint64_t*>(fring2 + NS * SLOT);
  const int nx = (int)op.nx, ny = (int)op.ny, nz = (int)op.nz;
  const int tx = threadIdx.x % TXP, ty = threadIdx.x / TXP;
  const int i = blockIdx.x * TX + 2 * tx;
  const int j = blockIdx.y * TY + ty;
  const bool in = i < nx && j < ny;
  const int l0 = blockIdx.z * kz, l1 = min(nz, l0 + kz);
  const int64_t plane = (int64_t)nx * ny;
  const double ch2 = op.ch2;
  const bool hW = in && i > 0, hE = in && i + 2 < nx, hS = in && j > 0, hN = in && j + 1 < ny;
  const bool needk = in && (i == 0 || j == 0);
  const int64_t c = in ? (int64_t)j * nx + i : 0;
  const double* col = x + c;
  const double* fx = op.faces + c;
  const double* fy = fx + op.n;
  const double* fz = fy + op.n;
  const double* kc_ = op.kcell + c;
  const int ox = (ty + 1) * XW + 2 + 2 * tx;
  const int ofx = OFX + ty * FXW + 2 + 2 * tx;
  const int ofy = OFY + (ty + 1) * TX + 2 * tx;
  const int ofz = OFZ + ty * TX + 2 * tx;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int qend = min(l1, nz - 1);  // last plane this CTA reads (x only when it is l1)
  const bool lead = threadIdx.x == 0;
  if (lead) {
#pragma unroll
    for (int st = 0; st < NS; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int p) {  // plane l0 + p into slot p % NS (the leader)
    const int q = l0 + p;
    if (q <= qend) {
      const int st = p % NS;
      double* sl = fring2 + st * SLOT;
      const bool faces = q < l1;
      mbar_arrive_expect_tx(&full[st], faces ? BX + BFX + BFY + BFZ : BX);
      tma_load_3d(sl, &tmx, i0 - 2, j0 - 1, q, &full[st]);
      if (faces) {
        tma_load_3d(sl + OFX, &tmfx, i0 - 2, j0, q, &full[st]);
        tma_load_3d(sl + OFY, &tmfy, i0, j0 - 1, q, &full[st]);
        tma_load_3d(sl + OFZ, &tmfz, i0, j0, q, &full[st]);
      }
    }
  };
  if (lead) {
#pragma unroll
    for (int p = 0; p < NS - 1; ++p) issue(p);
  }
  double2 xm = make_double2(0.0, 0.0), fzm = xm;
  if (in) {
    if (l0 > 0) {
      xm = *reinterpret_cast<const double2*>(col + (int64_t)(l0 - 1) * plane);
      fzm = *reinterpret_cast<const double2*>(fz + (int64_t)(l0 - 1) * plane);
    } else {
      fzm = *reinterpret_cast<const double2*>(kc_);  // own k on the domain boundary
    }
  }
  mbar_wait(&full[0], 0);
  int sc = 0, s1 = 1 % NS;
  uint32_t par1 = 0;  // parity of the phase plane p + 1 completes in its slot
  for (int l = l0; l < l1; ++l) {
    __syncthreads();  // everyone is done with plane p - 1: its slot takes plane p + NS - 1
    if (lead) issue(l - l0 + NS - 1);
    if (l + 1 < nz) mbar_wait(&full[s1], par1);
    if (in) {
      const double* sl = fring2 + sc * SLOT;
      const bool hZ = l + 1 < nz;
      double2 kc = make_double2(0.0, 0.0);
      if (needk) kc = *reinterpret_cast<const double2*>(kc_ + (int64_t)l * plane);
      const double2 C = *reinterpret_cast<const double2*>(sl + ox);
      const double2 fE = *reinterpret_cast<const double2*>(sl + ofx);
      const double2 fN = *reinterpret_cast<const double2*>(sl + ofy);
      const double2 fZ = *reinterpret_cast<const double2*>(sl + ofz);
      const double fW0 = hW ? sl[ofx - 1] : kc.x;
      const double fW1 = fE.x;  // (the pair's shared face)
      double2 fS = kc, S = make_double2(0.0, 0.0), N = S, Z = S;
      if (hS) {
        fS = *reinterpret_cast<const double2*>(sl + ofy - TX);
        S = *reinterpret_cast<const double2*>(sl + ox - XW);
      }
      if (hN) N = *reinterpret_cast<const double2*>(sl + ox + XW);
      if (hZ) Z = *reinterpret_cast<const double2*>(fring2 + s1 * SLOT + ox);
      double d0 = fzm.x, d1 = fzm.y;
      d0 = __dadd_rn(d0, fS.x);
      d1 = __dadd_rn(d1, fS.y);
      d0 = __dadd_rn(d0, fW0);
      d1 = __dadd_rn(d1, fW1);
      d0 = __dadd_rn(d0, fE.x);
      d1 = __dadd_rn(d1, fE.y);
      d0 = __dadd_rn(d0, fN.x);
      d1 = __dadd_rn(d1, fN.y);
      d0 = __dadd_rn(d0, fZ.x);
      d1 = __dadd_rn(d1, fZ.y);
      double a0 = 0.0, a1 = 0.0;
      if (l > 0) {
        a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fzm.x, ch2), xm.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fzm.y, ch2), xm.y));
      }
      if (hS) {
        a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fS.x, ch2), S.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fS.y, ch2), S.y));
      }
      if (hW) a0 = __dadd_rn(a0, __dmul_rn(__dsub_rn(-fW0, ch2), sl[ox - 1]));
      a1 = __dadd_rn(a1, __dmul_rn(__dsub_rn(-fW1, ch2), C.x));
      a0 = __dadd_rn(a0, __dmul_rn(d0, C.x));
      a1 = __dadd_rn(a1, __dmul_rn(d1, C.y));
      a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fE.x, ch2), C.y));
      if (hE) a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fE.y, ch2), sl[ox + 2]));
      if (hN) {
        a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fN.x, ch2), N.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fN.y, ch2), N.y));
      }
      if (hZ) {
        a0 = __dadd_rn(a0, __dmul_rn(__dadd_rn(-fZ.x, ch2), Z.x));
        a1 = __dadd_rn(a1, __dmul_rn(__dadd_rn(-fZ.y, ch2), Z.y));
      }
      *reinterpret_cast<double2*>(y + (int64_t)l * plane + c) = make_double2(a0, a1);
      xm = C;
      fzm = fZ;
    }
    sc = s1;
    s1 = s1 + 1 == NS ? 0 : s1 + 1;
    if (s1 == 0) par1 ^= 1u;
  }
}

// planes per CTA of the ring kernels.  A CTA walks one z chunk of one (x, y) tile; the chunks
// are sized so that the grid is a whole number of waves of resident CTAs, as nearly as the D + 2
// extra plane loads per chunk allow (256^3 with 16-plane chunks: 2.3 waves, i.e. a third wave at
// 31% -- measured 61 us; one wave of 43-plane chunks: 50 us)
static int ring_kz(const DevOp& op, int64_t tiles, int slots) {
  static const int kze = std::getenv("SKC_APPLY_KZ") ? std::atoi(std::getenv("SKC_APPLY_KZ")) : 0;
  if (kze > 0) return kze;
  int best_kz = (int)op.nz;
  double best = 0.0;
  for (int nch = 1; nch <= op.nz; ++nch) {
    const int kz = (int)((op.nz + nch - 1) / nch);
    if (kz < 12 && nch > 1) break;
    const int64_t w = tiles * ((op.nz + kz - 1) / kz);
    const double eff = (double)w / (double)(((w + slots - 1) / slots) * slots) * kz / (kz + 3.0);
    if (eff > best * 1.02) best = eff, best_kz = kz;  // (fewer, longer chunks unless clearly better)
  }
  return best_kz;
}

template <class K>
static int ring_slots(Ctx& c, K* kernel, size_t smem) {
  static int per_sm = 0;  // (per kernel instantiation; its callers pass one smem size each)
  static size_t for_smem = ~(size_t)0;
  if (for_smem != smem) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, smem));
    for_smem = smem;
  }
  return std::max(1, per_sm) * c.sm_count;
}

template <int D, int TY>
static void launch_apply3r2(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond) {
  constexpr int TX = 2 * (256 / TY);
  const size_t smem = sizeof(double) * (size_t)(D + 2) * (TY + 2) * (TX + 4);
  ensure_smem(k_apply3r2<D, TY>, smem);
  const int64_t tx = (op.nx + TX - 1) / TX, ty = (op.ny + TY - 1) / TY;
  const int kz = ring_kz(op, tx * ty, ring_slots(c, k_apply3r2<D, TY>, smem));
  const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
  launch_k(c, k_apply3r2<D, TY>, gr, 256, smem, op, x, y, kz, halt, cond);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

template <int NS, int R, bool DN = false, bool EF = false>
static bool launch_apply3t(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond) {
  static_assert(NS >= 3, "planes p, p + 1 are read while plane p + NS - 1 lands");
  using G = AtGeo<R>;
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)op.nx, (cuuint64_t)op.ny, (cuuint64_t)op.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)op.nx * 8, (cuuint64_t)op.nx * op.ny * 8};
  const cuuint32_t box[3] = {AT_W, G::H, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const size_t smem = sizeof(double) * (size_t)NS * G::SLOT + sizeof(uint64_t) * NS;
  ensure_smem(k_apply3t<NS, R, DN, EF>, smem);
  const int64_t tx = (op.nx + AT_TX - 1) / AT_TX, ty = (op.ny + G::TY - 1) / G::TY;
  const int kz = ring_kz(op, tx * ty, ring_slots(c, k_apply3t<NS, R, DN, EF>, smem));
  const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
  launch_k(c, k_apply3t<NS, R, DN, EF>, gr, 256, smem, tm, op, x, y, kz, halt, cond);
  return true;
}

static bool encode_map3(CUtensorMap* tm, const double* base, const DevOp& op, int bw, int bh) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)op.nx, (cuuint64_t)op.ny, (cuuint64_t)op.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)op.nx * 8, (cuuint64_t)op.nx * op.ny * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NS>
static bool launch_apply3t_face(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond) {
  static_assert(NS >= 3, "planes p, p + 1 are read while plane p + NS - 1 lands");
  using namespace fpt;
  if ((((uintptr_t)op.faces) & 15) != 0 || (op.n & 1)) return false;
  CUtensorMap tmx, tmfx, tmfy, tmfz;
  if (!encode_map3(&tmx, x, op, XW, XH) || !encode_map3(&tmfx, op.faces, op, FXW, TY) ||
      !encode_map3(&tmfy, op.faces + op.n, op, TX, TY + 1) || !encode_map3(&tmfz, op.faces + 2 * op.n, op, TX, TY))
    return false;
  const size_t smem = sizeof(double) * (size_t)NS * SLOT + sizeof(uint64_t) * NS;
  ensure_smem(k_apply3t_face<NS>, smem);
  const int64_t tx = (op.nx + TX - 1) / TX, ty = (op.ny + TY - 1) / TY;
  const int kz = ring_kz(op, tx * ty, ring_slots(c, k_apply3t_face<NS>, smem));
  const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
  launch_k(c, k_apply3t_face<NS>, gr, 256, smem, tmx, tmfx, tmfy, tmfz, op, x, y, kz, halt, cond);
  return true;
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
        if (c.apply_tma && c.apply_ring && op.nx % 2 == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0) {
          if (c.apply_alt && c.apply_tma == 3) {  // chained applies alternate their z direction (L2 reuse)
            c.apply_flip ^= 1;
            const bool ok = c.apply_alt == 2 ? (c.apply_flip ? launch_apply3t<3, 1, true, true>(c, op, x, y, halt, cond)
                                                             : launch_apply3t<3, 1, false, true>(c, op, x, y, halt, cond))
                                             : (c.apply_flip ? launch_apply3t<3, 1, true, false>(c, op, x, y, halt, cond)
                                                             : launch_apply3t<3, 1, false, false>(c, op, x, y, halt, cond));
            if (ok) break;
          }
          // SKC_APPLY_TMA = 10 * rows-per-thread + ring slots (a bare slot count means one row)
          const int ns = c.apply_tma % 10, rr = c.apply_tma / 10;
          const bool ok = rr == 2   ? (ns == 4 ? launch_apply3t<4, 2>(c, op, x, y, halt, cond)
                                               : launch_apply3t<3, 2>(c, op, x, y, halt, cond))
                          : rr == 4 ? (ns == 4 ? launch_apply3t<4, 4>(c, op, x, y, halt, cond)
                                               : launch_apply3t<3, 4>(c, op, x, y, halt, cond))
                          : ns == 4 ? launch_apply3t<4, 1>(c, op, x, y, halt, cond)
                          : ns == 6 ? launch_apply3t<6, 1>(c, op, x, y, halt, cond)
                          : ns == 8 ? launch_apply3t<8, 1>(c, op, x, y, halt, cond)
                                    : launch_apply3t<3, 1>(c, op, x, y, halt, cond);
          if (ok) break;
        }
        if (c.apply_ring && op.nx % 2 == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0) {
          static const int ty = std::getenv("SKC_APPLY_TY") ? std::atoi(std::getenv("SKC_APPLY_TY")) : 4;
          static const int dd = std::getenv("SKC_APPLY_D") ? std::atoi(std::getenv("SKC_APPLY_D")) : 1;
          if (ty == 4) {
            if (dd == 1)
              launch_apply3r2<1, 4>(c, op, x, y, halt, cond);
            else if (dd == 2)
              launch_apply3r2<2, 4>(c, op, x, y, halt, cond);
            else
              launch_apply3r2<4, 4>(c, op, x, y, halt, cond);
          } else {
            if (dd == 1)
              launch_apply3r2<1, 8>(c, op, x, y, halt, cond);
            else if (dd == 2)
              launch_apply3r2<2, 8>(c, op, x, y, halt, cond);
            else
              launch_apply3r2<4, 8>(c, op, x, y, halt, cond);
          }
          break;
        }
        if (c.apply_ring) {
          const int64_t tx = (op.nx + AR_TX - 1) / AR_TX, ty = (op.ny + AR_TY - 1) / AR_TY;
          const int kz = ring_kz(op, tx * ty, ring_slots(c, k_apply3r<4>, 0));
          const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
          launch_k(c, k_apply3r<4>, gr, AR_TX * AR_TY, 0, op, x, y, kz, halt, cond);
          break;
        }
        const dim3 gz((unsigned)((op.nx + AZ_TX - 1) / AZ_TX), (unsigned)((op.ny + AZ_TY - 1) / AZ_TY),
                      (unsigned)((op.nz + AZ_KZ - 1) / AZ_KZ));
        launch_k(c, k_apply3z, gz, AZ_TX * AZ_TY, 0, op, x, y, halt, cond);
        break;
      }
      case 32: {
        if (op.faces && c.apply_tma_face && c.apply_ring && op.nx % 2 == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0) {
          const bool ok = c.apply_tma_face == 4 ? launch_apply3t_face<4>(c, op, x, y, halt, cond)
                                                : launch_apply3t_face<3>(c, op, x, y, halt, cond);
          if (ok) break;
        }
        if (op.faces && c.apply_ring && op.nx % 2 == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0) {
          static const int dsel = std::getenv("SKC_APPLY_FD") ? std::atoi(std::getenv("SKC_APPLY_FD")) : 1;
          const int64_t tx = (op.nx + fp::TX - 1) / fp::TX, ty = (op.ny + fp::TY - 1) / fp::TY;
          auto go = [&](auto kern, int D) {
            const size_t smem = sizeof(double) * (size_t)(D + 2) * fp::SLOT;
            ensure_smem(kern, smem);
            const int kz = ring_kz(op, tx * ty, ring_slots(c, kern, smem));
            const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
            launch_k(c, kern, gr, 256, smem, op, x, y, kz, halt, cond);
          };
          if (dsel == 3)
            go(k_apply3r2_face<3>, 3);
          else if (dsel == 1)
            go(k_apply3r2_face<1>, 1);
          else
            go(k_apply3r2_face<2>, 2);
          break;
        }
        if (op.faces && c.apply_ring) {
          constexpr int D = 3;
          const size_t smem = sizeof(double) * (size_t)(D + 2) * AF2_SLOT;
          ensure_smem(k_apply3r_face<D>, smem);
          const int64_t tx = (op.nx + AR_TX - 1) / AR_TX, ty = (op.ny + AR_TY - 1) / AR_TY;
          const int kz = ring_kz(op, tx * ty, ring_slots(c, k_apply3r_face<D>, smem));
          const dim3 gr((unsigned)tx, (unsigned)ty, (unsigned)((op.nz + kz - 1) / kz));
          launch_k(c, k_apply3r_face<D>, gr, AR_TX * AR_TY, smem, op, x, y, kz, halt, cond);
          break;
        }
        if (op.faces) {
          const dim3 gf((unsigned)((op.nx + AF_TX - 1) / AF_TX), (unsigned)((op.ny + AF_TY - 1) / AF_TY),
                        (unsigned)((op.nz + AF_KZ - 1) / AF_KZ));
          launch_k(c, k_apply3z_face, gf, AF_TX * AF_TY, 0, op, x, y, halt, cond);
          break;
        }
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
