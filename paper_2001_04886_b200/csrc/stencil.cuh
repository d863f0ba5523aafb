// stencil.cuh -- one output point of the operators, bit-identical to the reference spmv
// (sparse.hpp:135-146): acc = 0, then + v*x per present neighbour / stored entry in ascending
// column order, multiply and add rounded separately.  Single-GPU geometry.
#pragma once

#include "skc_internal.hpp"

namespace skc {

__device__ __forceinline__ double face_k(double kp, double kq) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, kp), kq), __dadd_rn(kp, kq));
}

// x[q] is read through fetch(q) (a vector in memory, or a shared-memory slice with a
// fallback to memory outside it)
template <int DIM, int KIND, class F>
__device__ __forceinline__ double stencil_point_f(const DevOp& op, F&& fetch, int64_t i, int64_t j, int64_t l) {
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
    if (pres[t]) acc = __dadd_rn(acc, __dmul_rn(val[t], fetch(nb[t])));
  }
  return acc;
}

template <int DIM, int KIND>
__device__ __forceinline__ double stencil_point(const DevOp& op, const double* __restrict__ x, int64_t i,
                                                int64_t j, int64_t l) {
  return stencil_point_f<DIM, KIND>(op, [&](int64_t q) { return x[q]; }, i, j, l);
}

// grid coordinates of a point index walked with a fixed stride (no division per step)
struct GridWalk {
  int64_t i, j, l;
  __device__ __forceinline__ void init(const DevOp& op, int64_t p) {
    i = j = l = 0;
    if (op.kind == kCsr) return;  // (no grid)
    i = p % op.nx;
    j = (p / op.nx) % op.ny;
    l = p / (op.nx * op.ny);
  }
  __device__ __forceinline__ void step(const DevOp& op, int64_t stride) {
    if (op.kind == kCsr) return;
    i += stride;
    while (i >= op.nx) {
      i -= op.nx;
      if (++j == op.ny) j = 0, ++l;
    }
  }
};

// (A x)[p] at natural index p = (i, j, l) for any single-GPU operator, x read through fetch
template <class F>
__device__ __forceinline__ double apply_point(const DevOp& op, F&& fetch, int64_t p, const GridWalk& w) {
  if (op.kind == kCsr) {
    double acc = 0.0;
    for (int64_t q = op.rowptr[p]; q < op.rowptr[p + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(op.vals[q], fetch(op.colidx[q])));
    return acc;
  }
  const int64_t i = w.i, j = w.j, l = w.l;
  if (op.dim == 2) {
    if (op.kind == kStencilConst) return stencil_point_f<2, kStencilConst>(op, fetch, i, j, 0);
    if (op.kind == kStencilVarK) return stencil_point_f<2, kStencilVarK>(op, fetch, i, j, 0);
    return stencil_point_f<2, kStencilDia>(op, fetch, i, j, 0);
  }
  if (op.kind == kStencilConst) return stencil_point_f<3, kStencilConst>(op, fetch, i, j, l);
  if (op.kind == kStencilVarK) return stencil_point_f<3, kStencilVarK>(op, fetch, i, j, l);
  return stencil_point_f<3, kStencilDia>(op, fetch, i, j, l);
}

}  // namespace skc
