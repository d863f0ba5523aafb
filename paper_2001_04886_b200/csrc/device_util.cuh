// device_util.cuh -- device helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "skc_internal.hpp"

namespace skc {

// Non-contracted IEEE ops: the reference's y[i] += alpha * x[i] is a multiply then an add
// (no -march, no FMA; proj/CMakeLists.txt:6-8).  Every bit-exact (non-reduction) kernel
// goes through these.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool skip_launch(const int* halt, const int* cond) {
  if (halt && *(volatile const int*)halt) return true;
  if (cond && *(volatile const int*)cond == 0) return true;
  return false;
}

// Deterministic reduction of nd dots from per-CTA partials ([(d0+d)*G + g]) into out[d]
// (shared or global). Whole block must call; ends with __syncthreads().
__device__ __forceinline__ void reduce_dots_dev(const double* __restrict__ partials, int G, int d0, int nd,
                                                double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int d = warp; d < nd; d += nw) {
    const double* p = partials + (int64_t)(d0 + d) * G;
    double s = 0.0;
    for (int g = lane; g < G; g += 32) s += p[g];
    s = warp_sum(s);
    if (lane == 0) out[d] = s;
  }
  __syncthreads();
}

}  // namespace skc
