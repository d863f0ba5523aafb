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

// Kernel entry under programmatic dependent launch: release the next kernel on the stream for
// scheduling, then wait until the previous grid has completed and its memory is visible
// (both are no-ops for an ordinary launch).  Every kernel starts with this.
#define SKC_PDL_ENTRY()                                          \
  do {                                                           \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");              \
  } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp sums of K values at once: out[q] = sum over the 32 lanes of v[q] (q < K), written by
// one lane per value.  Recursive halving: at each of log2(P) exchange steps (P = K rounded up
// to a power of two, at most 32 per chunk) a lane keeps one half of its values and adds the
// partner's copy of that half, so the exchanges total ~P instead of 5K (one shuffle per value
// per level for a butterfly of each value); the remaining lane bits are then folded by plain
// butterflies.  Fixed order: deterministic.
template <int K>
__device__ __forceinline__ void warp_sums(const double (&acc)[K], double* out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c0 = 0; c0 < K; c0 += 32) {
    constexpr int CH = K < 32 ? K : 32;
    constexpr int P = CH <= 1 ? 1 : CH <= 2 ? 2 : CH <= 4 ? 4 : CH <= 8 ? 8 : CH <= 16 ? 16 : 32;
    constexpr int M = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : P == 8 ? 3 : P == 16 ? 4 : 5;
    double v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = c0 + q < K ? acc[c0 + q < K ? c0 + q : 0] : 0.0;
#pragma unroll
    for (int t = 0; t < M; ++t) {
      const int o = 16 >> t, h = P >> (t + 1);
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const double send = upper ? v[q] : v[q + h];
        const double keep = upper ? v[q + h] : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    double r = v[0];
#pragma unroll
    for (int o = (16 >> M); o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    const int idx = M == 0 ? 0 : lane >> (5 - M);
    if ((lane & ((1 << (5 - M)) - 1)) == 0 && c0 + idx < K) out[c0 + idx] = r;
  }
}

// The flags are written only by earlier kernels on the stream, so a read-only-path load is
// safe; it is served from L1 after the first warp per SM instead of serializing every warp
// of the grid on one L2 line.
__device__ __forceinline__ bool skip_launch(const int* halt, const int* cond) {
  if (halt && __ldg(halt)) return true;
  if (cond && __ldg(cond) == 0) return true;
  return false;
}

// ---------------------------------------------------------------- bulk async copies (TMA engine)
// cp.async.bulk global->shared with mbarrier completion (SASS UBLKCP / SYNCS): one elected
// thread arms the barrier with the expected byte count, lanes issue one copy per vector tile.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// one polling attempt (the producer of the block-iteration kernel also watches a quit flag)
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction-priority policies for cache-hinted loads/stores
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// per-thread asynchronous 8-byte global->shared copy (zero-fills when !pred); one commit
// group per call site step, waited with cp_async_wait<N> (N = groups allowed in flight)
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(pred ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Deterministic reduction of nd dots from per-CTA partials ([(d0+d)*G + g]) into out[d]
// (shared or global). Whole block must call; ends with __syncthreads().
// Each dot is owned by a group of TPD lanes (TPD = 32 >> k, chosen so all dots are covered
// in few rounds); every lane sums a fixed strided subset with four independent accumulators
// (loads stay in flight), then the group combines in a fixed shuffle order.
// Grouped partials (G >> 16 = cpg, Geo::enc): sum every group's cpg partials in order, then the
// group sums in order -- a fixed tree whatever the GPU count (reduce_point allgathers the group
// sums across ranks and passes them on with cpg = 1).  One warp per dot.
__device__ __forceinline__ void reduce_dots_grouped(const double* __restrict__ partials, int G, int d0, int nd,
                                                    double* out) {
  const int Gn = G & 0xffff, cpg = G >> 16, ngrp = Gn / cpg;
  const int lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int d = threadIdx.x >> 5; d < nd; d += nwarp) {
    const double* p = partials + (int64_t)(d0 + d) * kPartialPitch;
    double gs[2] = {0.0, 0.0};  // groups lane and lane + 32 (at most 64 groups)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int grp = lane + 32 * h;
      if (grp < ngrp) {
        double a = 0.0;
        for (int j = 0; j < cpg; ++j) a += p[grp * cpg + j];
        gs[h] = a;
      }
    }
    double tot = 0.0;
    for (int grp = 0; grp < ngrp; ++grp) tot += __shfl_sync(0xffffffffu, (grp >> 5) ? gs[1] : gs[0], grp & 31);
    if (lane == 0) out[d] = tot;
  }
  __syncthreads();
}

__device__ __forceinline__ void reduce_dots_dev(const double* __restrict__ partials, int G, int d0, int nd,
                                                double* out) {
  if (G >> 16) {
    reduce_dots_grouped(partials, G, d0, nd, out);
    return;
  }
  const int nthreads = blockDim.x;
  int tpd = 32;
  while (tpd > 1 && (nthreads / tpd) < nd) tpd >>= 1;
  const int groups = nthreads / tpd;
  const int grp = threadIdx.x / tpd, sub = threadIdx.x % tpd;
  for (int d = grp; d - grp < nd; d += groups) {  // uniform trip count across the warp
    double s = 0.0;
    if (d < nd) {
      const double* p = partials + (int64_t)(d0 + d) * kPartialPitch;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int g = sub;
#pragma unroll 4
      for (; g + 3 * tpd < G; g += 4 * tpd) {
        a0 += p[g];
        a1 += p[g + tpd];
        a2 += p[g + 2 * tpd];
        a3 += p[g + 3 * tpd];
      }
      for (; g < G; g += tpd) a0 += p[g];
      s = (a0 + a1) + (a2 + a3);
    }
    for (int o = tpd >> 1; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, tpd);
    if (sub == 0 && d < nd) out[d] = s;
  }
  __syncthreads();
}

}  // namespace skc
