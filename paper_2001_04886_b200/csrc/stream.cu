// stream.cu -- the streaming kernels every solver phase is built from.  Input tiles are
// staged through shared memory by the bulk-copy (TMA) engine in a warp-specialized
// producer/consumer pipeline:
//
//   producer warp : for each tile of T points, waits until its stage is free (empty
//                   mbarrier), arms the stage's full mbarrier with the byte count and issues
//                   one cp.async.bulk per distinct operand vector;
//   consumer warps: wait on the full mbarrier, compute from shared memory, and release the
//                   stage with one arrive per warp -- no CTA-wide barrier per tile.
//
// Kernels:
//  * k_upd<NOUT, MAXD, PPT> : generic fused block vector update y_o = base_o [* c] +
//        sum_j c_{j,o} x_j in the reference's per-element order (axpy / block_axpy_inplace,
//        kernels.hpp:55-58, block.hpp:109-116; multiply and add rounded separately) plus up
//        to MAXD inner products of the results (deterministic per-CTA partials).
//  * k_mgs<S, DOTS> : one block-MGS round of s-step Arnoldi (sstep.hpp:346-352),
//        cand[:,jc] -= sum_l t(l,jc-1) V_i[:,l], fused with the next round's
//        V_{i+1}^T cand products (sstep.hpp:341), everything compile-time sized.
//  * k_grm<NR, LB> : packed block inner products L^T R (block_gram / block_dot,
//        block.hpp:70-99).
#include <algorithm>
#include <cstring>

#include "device_util.cuh"
#include "skc_internal.hpp"

namespace skc {

namespace {

constexpr int kMaxStage = 4;
constexpr int NCW = 8;                  // consumer warps
constexpr int CONS = NCW * 32;          // consumer threads
constexpr int THREADS = CONS + 32;      // + one producer warp
constexpr int UPD_MAXU = LC_MAXOUT + LC_MAXIN + LC_MAXX;
constexpr int GRM_MAXU = GR_MAXL + GR_MAXR;

// common pipeline header of every descriptor
struct PipeHdr {
  int nu, T, nstage;
  int64_t n, range;
  int cpg;
  int64_t gsize;
  const int* halt;
  const int* cond;
};

struct UpdDesc {
  PipeHdr h;
  int nin, nout, nx, nd, ncoef;
  int nin0;  // SPLIT: terms [0, nin0) feed outputs [0, NOUT/2), the rest [NOUT/2, NOUT)
  const double* U[UPD_MAXU];  // distinct staged vectors
  uint8_t ub[LC_MAXOUT];      // base of output q -> U index
  int16_t bscale[LC_MAXOUT];
  double* out[LC_MAXOUT];
  uint8_t ut[LC_MAXIN];  // term j -> U index
  uint16_t mask[LC_MAXIN];
  int16_t cbase[LC_MAXIN];
  uint8_t ux[LC_MAXX];  // extra x -> U index
  uint8_t da[LC_MAXD], db[LC_MAXD];
  const double* coef;
  double* partials;
  int dot0, G;
};

struct GrmDesc {
  PipeHdr h;
  int nl, nr;
  const double* U[GRM_MAXU];
  uint8_t li[GR_MAXL], ri[GR_MAXR];
  double* partials;
  int G;
  int rbase[GR_MAXR], rstride[GR_MAXR], lmax[GR_MAXR];  // output map (see GramDesc)
};

struct MgsDesc {
  PipeHdr h;
  const double* U[3 * kMaxS];  // V_i[0..S), cand[1..S), V_{i+1}[0..S) (DOTS)
  double* cand[kMaxS];         // outputs cand[1..S)
  MgsScalar sc;                // the round's scalar step (prologue)
  double* partials;
  int dot0, G;
};

struct TileGeom {
  int64_t start;
  int cnt;
  bool bulk;
};
__device__ __forceinline__ TileGeom tile_geom(const PipeHdr& h, int64_t r0, int64_t r1, int t) {
  TileGeom g;
  g.start = r0 + (int64_t)t * h.T;
  g.cnt = (int)(r1 - g.start < (int64_t)h.T ? r1 - g.start : (int64_t)h.T);
  g.bulk = ((g.cnt | (int)g.start) & 1) == 0;  // bulk copies move 16-byte-aligned multiples of 16 bytes
  return g;
}

struct Pipe {
  uint64_t* full;
  uint64_t* empty;
  double* stages;
  size_t stage_sz;
  int64_t r0, r1;
  int ntiles;
};

__device__ __forceinline__ Pipe pipe_setup(const PipeHdr& h, unsigned char* smem_raw, size_t prefix_bytes) {
  Pipe p;
  p.full = reinterpret_cast<uint64_t*>(smem_raw);
  p.empty = p.full + kMaxStage;
  p.stages = reinterpret_cast<double*>(smem_raw + 64 + prefix_bytes);
  p.stage_sz = (size_t)h.nu * h.T;
  {  // (grouped geometry: CTA b is member b % cpg of group b / cpg)
    const int64_t grp = blockIdx.x / h.cpg, mem = blockIdx.x % h.cpg;
    p.r0 = grp * h.gsize + mem * h.range;
    p.r1 = min(min(h.n, (grp + 1) * h.gsize), p.r0 + h.range);
  }
  p.ntiles = p.r1 > p.r0 ? (int)((p.r1 - p.r0 + h.T - 1) / h.T) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < h.nstage; ++s) {
      mbar_init(&p.full[s], 1);
      mbar_init(&p.empty[s], NCW);
    }
    mbar_fence_init();
  }
  return p;
}

// producer warp: stream every tile of this CTA's range through the stages
template <int MAXU>
__device__ __forceinline__ void pipe_produce(const PipeHdr& h, const double* const (&U)[MAXU], const Pipe& p,
                                             int t0 = 0, int t1 = -1) {
  const int lane = threadIdx.x & 31;
  if (t1 < 0 || t1 > p.ntiles) t1 = p.ntiles;
  for (int t = t0; t < t1; ++t) {
    const int st = t % h.nstage, u = t / h.nstage;
    if (u > 0) mbar_wait(&p.empty[st], (uint32_t)((u - 1) & 1));
    const TileGeom g = tile_geom(h, p.r0, p.r1, t);
    double* S = p.stages + (size_t)st * p.stage_sz;
    if (g.bulk) {
      const uint32_t bytes = (uint32_t)g.cnt * 8u;
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&p.full[st], bytes * (uint32_t)h.nu);
      }
      __syncwarp();
      for (int v = lane; v < h.nu; v += 32) bulk_g2s(S + (size_t)v * h.T, U[v] + g.start, bytes, &p.full[st]);
    } else {
      for (int v = 0; v < h.nu; ++v)
        for (int q = lane; q < g.cnt; q += 32) S[(size_t)v * h.T + q] = U[v][g.start + q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&p.full[st]);
    }
  }
}

__device__ __forceinline__ double* pipe_acquire(const PipeHdr& h, const Pipe& p, int t, TileGeom& g) {
  const int st = t % h.nstage;
  mbar_wait(&p.full[st], (uint32_t)((t / h.nstage) & 1));
  g = tile_geom(h, p.r0, p.r1, t);
  return p.stages + (size_t)st * p.stage_sz;
}

__device__ __forceinline__ void pipe_release(const PipeHdr& h, const Pipe& p, int t) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&p.empty[t % h.nstage]);
}

// fixed-order CTA reduction of per-thread accumulators (consumer threads only hold data;
// all THREADS threads must call).  red: >= NCW * K doubles of shared memory.
template <int K>
__device__ __forceinline__ void cta_store_partials(const double (&acc)[K], int nk, double* red, double* partials,
                                                   int dot0, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp < NCW) warp_sums(acc, red + warp * K);  // (values k >= nk are summed but unused)
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < NCW; ++w) s += red[w * K + k];
    partials[(int64_t)(dot0 + k) * kPartialPitch + blockIdx.x] = s;
  }
}

// ------------------------------------------------------------------ k_upd
template <int NOUT, int MAXD, int PPT, bool SPLIT>
__global__ void __launch_bounds__(THREADS) k_upd(const __grid_constant__ UpdDesc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int coef_slots = (d.ncoef + 15) & ~15;
  // per-thread value columns for the fused products: the outputs, then the nx extra inputs
  const size_t prefix = 8 * ((size_t)coef_slots + (MAXD > 0 ? (size_t)(NOUT + d.nx) * CONS : 0));
  Pipe p = pipe_setup(d.h, smem_raw, prefix);
  double* scoef = reinterpret_cast<double*>(smem_raw + 64);
  double* sv = scoef + coef_slots;
  for (int t = threadIdx.x; t < d.ncoef; t += blockDim.x) scoef[t] = d.coef[t];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double acc[MAXD > 0 ? MAXD : 1];
#pragma unroll
  for (int k = 0; k < (MAXD > 0 ? MAXD : 1); ++k) acc[k] = 0.0;

  if (warp == NCW) {
    pipe_produce(d.h, d.U, p);
  } else {
    double* col = sv + threadIdx.x;
    const int T = d.h.T;
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      const double* S = pipe_acquire(d.h, p, t, g);
      const int p0 = threadIdx.x;
      if (p0 < g.cnt) {
        bool ok[PPT];
#pragma unroll
        for (int u = 0; u < PPT; ++u) ok[u] = p0 + CONS * u < g.cnt;
        double o[PPT][NOUT];
#pragma unroll
        for (int q = 0; q < NOUT; ++q) {
          const double* bq = S + (size_t)d.ub[q] * T + p0;
          const int bs = d.bscale[q];
          const double sc = bs >= 0 ? scoef[bs] : 1.0;
#pragma unroll
          for (int u = 0; u < PPT; ++u) {
            const double b = bq[CONS * u];
            o[u][q] = bs >= 0 ? dmul(b, sc) : b;
          }
        }
        if (SPLIT) {
          // two output halves, each fed by its own run of terms (term order within a half is
          // the reference's order for each of its outputs)
          constexpr int H = NOUT / 2;
          for (int j = 0; j < d.nin; ++j) {
            const double* vj = S + (size_t)d.ut[j] * T + p0;
            const double* cj = scoef + d.cbase[j];
            double v[PPT];
#pragma unroll
            for (int u = 0; u < PPT; ++u) v[u] = vj[CONS * u];
            if (j < d.nin0) {
#pragma unroll
              for (int q = 0; q < H; ++q) {
                const double c = cj[q];
#pragma unroll
                for (int u = 0; u < PPT; ++u) o[u][q] = dadd(o[u][q], dmul(c, v[u]));
              }
            } else {
#pragma unroll
              for (int q = H; q < NOUT; ++q) {
                const double c = cj[q];
#pragma unroll
                for (int u = 0; u < PPT; ++u) o[u][q] = dadd(o[u][q], dmul(c, v[u]));
              }
            }
          }
        }
        for (int j = 0; j < (SPLIT ? 0 : d.nin); ++j) {
          const double* vj = S + (size_t)d.ut[j] * T + p0;
          const unsigned m = d.mask[j];
          const double* cj = scoef + d.cbase[j];
          double v[PPT];
#pragma unroll
          for (int u = 0; u < PPT; ++u) v[u] = vj[CONS * u];
          if (NOUT == 1 || m == (1u << NOUT) - 1u) {  // dense term (all outputs): no predication
#pragma unroll
            for (int q = 0; q < NOUT; ++q) {
              const double c = cj[q];
#pragma unroll
              for (int u = 0; u < PPT; ++u) o[u][q] = dadd(o[u][q], dmul(c, v[u]));
            }
          } else {
#pragma unroll
            for (int q = 0; q < NOUT; ++q)
              if ((m >> q) & 1u) {
                const double c = cj[q];
#pragma unroll
                for (int u = 0; u < PPT; ++u) o[u][q] = dadd(o[u][q], dmul(c, v[u]));
              }
          }
        }
#pragma unroll
        for (int q = 0; q < NOUT; ++q) {
          double* oq = d.out[q] + g.start + p0;
#pragma unroll
          for (int u = 0; u < PPT; ++u)
            if (ok[u]) oq[CONS * u] = o[u][q];
        }
        if (MAXD > 0) {
#pragma unroll
          for (int u = 0; u < PPT; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int q = 0; q < NOUT; ++q) col[q * CONS] = o[u][q];
            for (int x = 0; x < d.nx; ++x) col[(NOUT + x) * CONS] = S[(size_t)d.ux[x] * T + p0 + CONS * u];
#pragma unroll
            for (int k = 0; k < (MAXD > 0 ? MAXD : 1); ++k)
              if (k < d.nd) acc[k] = fma(col[d.da[k] * CONS], col[d.db[k] * CONS], acc[k]);
          }
        }
      }
      pipe_release(d.h, p, t);
    }
  }
  if (MAXD > 0) cta_store_partials(acc, d.nd, sv, d.partials, d.dot0, d.G);
}

// ------------------------------------------------------------------ k_bupd
// The s-Omin direction-block update at s > 4 (sstep.hpp:215-222), one half (P or AP) per
// launch: S outputs y_q = base_q + sum_j c[j][q] x_j, every term dense, the coefficients one
// contiguous [nin][S] array, plus (DOTS) the upper triangle of the outputs' Gram matrix and
// their products with one extra vector (W and m).  k_upd walks a descriptor per term and spills
// its 64 product accumulators (C5: 2.9 TB/s); here the shape is compile time: the term loop is
// unrolled a block of S at a time with immediate stage offsets, the coefficients come as
// 16-byte broadcast loads and the products accumulate in registers straight from the outputs.
// Per-element order (multiply and add rounded separately, terms ascending) is k_upd's.
struct BupdDesc {
  PipeHdr h;
  int nin, cb0;
  const double* U[UPD_MAXU];  // [0,S) bases | [S, S+nin) terms | (DOTS) the extra vector
  double* out[kMaxS];
  const double* coef;
  double* partials;
  int dot0, G;
};

constexpr int BUPD_T = 2 * CONS;  // points per tile: two per consumer thread

template <int S, bool DOTS>
__global__ void __launch_bounds__(THREADS) k_bupd(const __grid_constant__ BupdDesc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int T = BUPD_T;
  constexpr int ND = DOTS ? S * (S + 1) / 2 + S : 1;
  const int coef_slots = (d.nin * S + 15) & ~15;
  const size_t prefix = 8 * ((size_t)coef_slots + (DOTS ? (size_t)NCW * ND : 0));
  Pipe p = pipe_setup(d.h, smem_raw, prefix);
  double* scoef = reinterpret_cast<double*>(smem_raw + 64);
  double* red = scoef + coef_slots;
  for (int t = threadIdx.x; t < d.nin * S; t += blockDim.x) scoef[t] = d.coef[d.cb0 + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double acc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) acc[k] = 0.0;

  if (warp == NCW) {
    pipe_produce(d.h, d.U, p);
  } else {
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      const double* St = pipe_acquire(d.h, p, t, g);
      const int p0 = threadIdx.x;
      if (p0 < g.cnt) {
        const bool ok1 = p0 + CONS < g.cnt;  // (the second point of a short tile: computed on stale data, not used)
        const double* sp = St + p0;
        double o0[S], o1[S];
#pragma unroll
        for (int q = 0; q < S; ++q) {
          o0[q] = sp[q * T];
          o1[q] = sp[q * T + CONS];
        }
        for (int j0 = 0; j0 < d.nin; j0 += S) {
          const double* x = sp + (size_t)(S + j0) * T;
          const double* cj = scoef + j0 * S;
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double v0 = x[l * T], v1 = x[l * T + CONS];
            double c[S];
            if constexpr (S % 2 == 0) {
#pragma unroll
              for (int q = 0; q < S; q += 2) {
                const double2 cc = *reinterpret_cast<const double2*>(cj + l * S + q);
                c[q] = cc.x;
                c[q + 1] = cc.y;
              }
            } else {
#pragma unroll
              for (int q = 0; q < S; ++q) c[q] = cj[l * S + q];
            }
#pragma unroll
            for (int q = 0; q < S; ++q) {
              o0[q] = dadd(o0[q], dmul(c[q], v0));
              o1[q] = dadd(o1[q], dmul(c[q], v1));
            }
          }
        }
        const int64_t at = g.start + p0;
#pragma unroll
        for (int q = 0; q < S; ++q) {
          d.out[q][at] = o0[q];
          if (ok1) d.out[q][at + CONS] = o1[q];
        }
        if (DOTS) {
          const double* xr = sp + (size_t)(S + d.nin) * T;
          const double r0 = xr[0];
          double r1 = xr[CONS];
          if (!ok1) {
            r1 = 0.0;
#pragma unroll
            for (int q = 0; q < S; ++q) o1[q] = 0.0;
          }
          int k = 0;
#pragma unroll
          for (int a = 0; a < S; ++a)
#pragma unroll
            for (int b = a; b < S; ++b, ++k) acc[k] = fma(o1[a], o1[b], fma(o0[a], o0[b], acc[k]));
#pragma unroll
          for (int a = 0; a < S; ++a, ++k) acc[k] = fma(o1[a], r1, fma(o0[a], r0, acc[k]));
        }
      }
      pipe_release(d.h, p, t);
    }
  }
  if (DOTS) cta_store_partials(acc, ND, red, d.partials, d.dot0, d.G);
}

// The fused form for s <= 4 (one launch for both halves, which share the powers block): outputs
// [P_0..P_{S-1}, AP_0..AP_{S-1}], term blocks [P_e columns, AP_e columns] per window block e, both
// halves with the same coefficients c[e][l][q]; products = the upper triangle of AP^T AP and AP^T x.
struct Bupd2Desc {
  PipeHdr h;
  int nin, cb0, nb0, ix;      // terms, coefficient offset, distinct base vectors, stage slot of the extra vector
  const double* U[UPD_MAXU];  // [0,nb0) bases | [nb0, nb0+nin) terms | (the extra vector, unless it is a base)
  uint8_t ub[2 * 4];          // base of output q -> stage slot
  double* out[2 * 4];
  const double* coef;
  double* partials;
  int dot0, G;
};

template <int S>
__global__ void __launch_bounds__(THREADS) k_bupd2(const __grid_constant__ Bupd2Desc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int T = BUPD_T, NO = 2 * S;
  constexpr int ND = S * (S + 1) / 2 + S;
  const int ncf = (d.nin / 2) * S;
  const int coef_slots = (ncf + 15) & ~15;
  const size_t prefix = 8 * ((size_t)coef_slots + (size_t)NCW * ND);
  Pipe p = pipe_setup(d.h, smem_raw, prefix);
  double* scoef = reinterpret_cast<double*>(smem_raw + 64);
  double* red = scoef + coef_slots;
  for (int t = threadIdx.x; t < ncf; t += blockDim.x) scoef[t] = d.coef[d.cb0 + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double acc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) acc[k] = 0.0;

  if (warp == NCW) {
    pipe_produce(d.h, d.U, p);
  } else {
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      const double* St = pipe_acquire(d.h, p, t, g);
      const int p0 = threadIdx.x;
      if (p0 < g.cnt) {
        const bool ok1 = p0 + CONS < g.cnt;
        const double* sp = St + p0;
        double o0[NO], o1[NO];
#pragma unroll
        for (int q = 0; q < NO; ++q) {
          const double* b = sp + (int)d.ub[q] * T;
          o0[q] = b[0];
          o1[q] = b[CONS];
        }
        for (int j0 = 0; j0 < d.nin; j0 += NO) {
          const double* x = sp + (size_t)(d.nb0 + j0) * T;
          const double* cj = scoef + (j0 / 2) * S;
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double vp0 = x[l * T], vp1 = x[l * T + CONS];
            const double va0 = x[(S + l) * T], va1 = x[(S + l) * T + CONS];
            double c[S];
            if constexpr (S % 2 == 0) {
#pragma unroll
              for (int q = 0; q < S; q += 2) {
                const double2 cc = *reinterpret_cast<const double2*>(cj + l * S + q);
                c[q] = cc.x;
                c[q + 1] = cc.y;
              }
            } else {
#pragma unroll
              for (int q = 0; q < S; ++q) c[q] = cj[l * S + q];
            }
#pragma unroll
            for (int q = 0; q < S; ++q) {
              o0[q] = dadd(o0[q], dmul(c[q], vp0));
              o1[q] = dadd(o1[q], dmul(c[q], vp1));
              o0[S + q] = dadd(o0[S + q], dmul(c[q], va0));
              o1[S + q] = dadd(o1[S + q], dmul(c[q], va1));
            }
          }
        }
        const int64_t at = g.start + p0;
#pragma unroll
        for (int q = 0; q < NO; ++q) {
          d.out[q][at] = o0[q];
          if (ok1) d.out[q][at + CONS] = o1[q];
        }
        const double* xr = sp + (size_t)d.ix * T;
        const double r0 = xr[0];
        double r1 = xr[CONS];
        if (!ok1) {
          r1 = 0.0;
#pragma unroll
          for (int q = 0; q < S; ++q) o1[S + q] = 0.0;
        }
        int k = 0;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int b = a; b < S; ++b, ++k) acc[k] = fma(o1[S + a], o1[S + b], fma(o0[S + a], o0[S + b], acc[k]));
#pragma unroll
        for (int a = 0; a < S; ++a, ++k) acc[k] = fma(o1[S + a], r1, fma(o0[S + a], r0, acc[k]));
      }
      pipe_release(d.h, p, t);
    }
  }
  cta_store_partials(acc, ND, red, d.partials, d.dot0, d.G);
}

// ------------------------------------------------------------------ k_mgs
// The round's scalar step (see launch_mgs): every CTA reduces the incoming products in the
// same fixed order and solves the same s x s system, so all CTAs apply identical t.  Whole
// block calls; coefficients -t land in cs[l*(S-1) + jc-1].
constexpr int kGramWords = (int)((sizeof(Gram) + 7) / 8);
// coefficients, products, Gram copy; a multiple of 128 bytes so the stages stay aligned
constexpr int kMgsPrefix = (8 * (64 + 64 + kGramWords) + 127) / 128 * 128;

template <int S>
__device__ __forceinline__ void mgs_scalar(const MgsScalar& sc, double* cs, double* tmp, Gram* gs) {
  constexpr int NC = S - 1;
  {  // stage block i's factor in shared memory: the serial solve then reads it at smem latency
    const uint64_t* src = reinterpret_cast<const uint64_t*>(sc.gram);
    uint64_t* dst = reinterpret_cast<uint64_t*>(gs);
    for (int w = threadIdx.x; w < (int)(sizeof(Gram) / 8); w += blockDim.x) dst[w] = src[w];
  }
  reduce_dots_dev(sc.src, sc.src_G, sc.src_d0, sc.full ? S * S : S * NC, tmp);  // ends with __syncthreads
  if (threadIdx.x < NC) {
    const int jc = threadIdx.x;
    double rhs[kMaxS], t[kMaxS];
#pragma unroll
    for (int l = 0; l < S; ++l) rhs[l] = sc.full ? tmp[l * S + jc + 1] : tmp[l * NC + jc];
    gram_solve_dev(*gs, rhs, t);
#pragma unroll
    for (int l = 0; l < S; ++l) {
      cs[l * NC + jc] = -t[l];
      if (blockIdx.x == 0) {
        double* ta = sc.rec_t + l * S + (jc + 1);
        *ta = sc.accumulate ? *ta + t[l] : t[l];
      }
    }
  }
  __syncthreads();
}

// The producer warp puts the first stages in flight before the scalar step so the tile loads
// overlap the reduction.
// U layout: [0,S) V_i ; [S, 2S-1) cand[1..S-1] ; [2S-1, 3S-1) V_{i+1} (DOTS)
template <int S, bool DOTS>
__global__ void __launch_bounds__(THREADS) k_mgs(const __grid_constant__ MgsDesc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NC = S - 1;
  constexpr int ND = DOTS ? S * NC : 1;
  Pipe p = pipe_setup(d.h, smem_raw, kMgsPrefix);
  double* red = reinterpret_cast<double*>(smem_raw + 64);  // 64 coefficients + 64 scratch doubles
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp == NCW) pipe_produce(d.h, d.U, p, 0, d.h.nstage);
  mgs_scalar<S>(d.sc, red, red + 64, reinterpret_cast<Gram*>(red + 128));
  // coefficients in registers for small S; for S >= 6 they are re-read from shared memory
  // (warp-uniform broadcast) to keep the accumulators in registers
  constexpr bool CREG = S < 6;
  double c[CREG ? S : 1][CREG ? NC : 1];
  if (CREG) {
#pragma unroll
    for (int l = 0; l < (CREG ? S : 1); ++l)
#pragma unroll
      for (int j = 0; j < (CREG ? NC : 1); ++j) c[l][j] = red[l * NC + j];
  }
  const double* cs = red;
  double acc[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) acc[k] = 0.0;
  if (warp == NCW) {
    pipe_produce(d.h, d.U, p, d.h.nstage);
  } else {
    const int T = d.h.T;
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      const double* Sm = pipe_acquire(d.h, p, t, g);
      for (int q = threadIdx.x; q < g.cnt; q += CONS) {
        double cv[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) cv[j] = Sm[(size_t)(S + j) * T + q];
#pragma unroll
        for (int l = 0; l < S; ++l) {
          const double v = Sm[(size_t)l * T + q];
#pragma unroll
          for (int j = 0; j < NC; ++j) cv[j] = dadd(cv[j], dmul(CREG ? c[CREG ? l : 0][CREG ? j : 0] : cs[l * NC + j], v));
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) d.cand[j][g.start + q] = cv[j];
        if (DOTS) {
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double w = Sm[(size_t)(2 * S - 1 + l) * T + q];
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[l * NC + j] = fma(w, cv[j], acc[l * NC + j]);
          }
        }
      }
      pipe_release(d.h, p, t);
    }
  }
  if (DOTS) {
    __syncthreads();  // coefficient area is reused for the reduction below
    cta_store_partials(acc, ND, p.stages, d.partials, d.dot0, d.G);
  }
}

// Two-phase variant for S >= 6, where S(S-1) per-thread accumulators would spill: the tile's
// new candidate columns are written back into their stage slots, the consumer warps meet at a
// named barrier, and the products with V_{i+1} are taken from shared memory with one warp per
// V_{i+1} column (S-1 accumulators per thread).  Partial layout as in k_mgs.
template <int S>
__global__ void __launch_bounds__(THREADS) k_mgs2(const __grid_constant__ MgsDesc d) {
  SKC_PDL_ENTRY();
  static_assert(S <= NCW, "one warp per V_{i+1} column");
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NC = S - 1;
  Pipe p = pipe_setup(d.h, smem_raw, kMgsPrefix);
  double* cs = reinterpret_cast<double*>(smem_raw + 64);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp == NCW) pipe_produce(d.h, d.U, p, 0, d.h.nstage);
  mgs_scalar<S>(d.sc, cs, cs + 64, reinterpret_cast<Gram*>(cs + 128));
  const bool dotw = warp < S;  // warp l owns the products with V_{i+1}[:, l]
  double acc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) acc[k] = 0.0;
  if (warp == NCW) {
    pipe_produce(d.h, d.U, p, d.h.nstage);
  } else {
    const int T = d.h.T;
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      double* Sm = pipe_acquire(d.h, p, t, g);
      for (int q = threadIdx.x; q < g.cnt; q += CONS) {
        double cv[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) cv[j] = Sm[(size_t)(S + j) * T + q];
#pragma unroll
        for (int l = 0; l < S; ++l) {
          const double v = Sm[(size_t)l * T + q];
#pragma unroll
          for (int j = 0; j < NC; ++j) cv[j] = dadd(cv[j], dmul(cs[l * NC + j], v));
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          d.cand[j][g.start + q] = cv[j];
          Sm[(size_t)(S + j) * T + q] = cv[j];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CONS) : "memory");
      if (dotw) {
        const double* wl = Sm + (size_t)(2 * S - 1 + warp) * T;
        for (int q = lane; q < g.cnt; q += 32) {
          const double w = wl[q];
#pragma unroll
          for (int j = 0; j < NC; ++j) acc[j] = fma(w, Sm[(size_t)(S + j) * T + q], acc[j]);
        }
      }
      fence_proxy_async();  // generic writes to the stage before the producer's next bulk copy
      pipe_release(d.h, p, t);
    }
  }
  __syncthreads();
  if (dotw) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const double v = warp_sum(acc[j]);
      if (lane == 0) d.partials[(int64_t)(d.dot0 + warp * NC + j) * kPartialPitch + blockIdx.x] = v;
    }
  }
}

// ------------------------------------------------------------------ k_grm
template <int NR, int LB>
__global__ void __launch_bounds__(THREADS) k_grm(const __grid_constant__ GrmDesc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.h.halt, d.h.cond)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Pipe p = pipe_setup(d.h, smem_raw, 0);
  __syncthreads();
  const int nch = (d.nl + LB - 1) / LB;  // <= NCW
  const int PG = max(1, NCW / nch);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int chunk = warp % nch, group = warp / nch;
  const bool active = warp < NCW && group < PG;
  const int l0 = chunk * LB;
  const int nlb = min(LB, d.nl - l0);
  constexpr int K = LB * NR;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;

  if (warp == NCW) {
    pipe_produce(d.h, d.U, p);
  } else {
    const int T = d.h.T;
    int ri[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) ri[r] = d.ri[r] * T;
    int li[LB];
#pragma unroll
    for (int lb = 0; lb < LB; ++lb) li[lb] = d.li[l0 + (lb < nlb ? lb : 0)] * T;
    for (int t = 0; t < p.ntiles; ++t) {
      TileGeom g;
      const double* Sm = pipe_acquire(d.h, p, t, g);
      if (active) {
        for (int q = group * 32 + lane; q < g.cnt; q += 32 * PG) {
          double rv[NR];
#pragma unroll
          for (int r = 0; r < NR; ++r) rv[r] = Sm[ri[r] + q];
#pragma unroll
          for (int lb = 0; lb < LB; ++lb) {
            const double lv = Sm[li[lb] + q];  // rows past nl duplicate row 0; discarded below
#pragma unroll
            for (int r = 0; r < NR; ++r) acc[lb * NR + r] = fma(lv, rv[r], acc[lb * NR + r]);
          }
        }
      }
      pipe_release(d.h, p, t);
    }
  }
  __syncthreads();
  double* red = p.stages;  // [group][chunk][K]
  if (active) warp_sums(acc, red + ((size_t)group * nch + chunk) * K);
  __syncthreads();
  for (int e = threadIdx.x; e < nch * K; e += blockDim.x) {
    const int ch = e / K, k = e % K, lb = k / NR, r = k % NR;
    const int l = ch * LB + lb;
    if (l < d.nl && l < d.lmax[r]) {  // rows past nl in the last chunk duplicated row 0: discarded
      double s = 0.0;
      for (int gp = 0; gp < PG; ++gp) s += red[((size_t)gp * nch + ch) * K + k];
      d.partials[(int64_t)(d.rbase[r] + l * d.rstride[r]) * kPartialPitch + blockIdx.x] = s;
    }
  }
}

// ------------------------------------------------------------------ host side
struct TileChoice {
  int T, nstage;
  size_t smem;
};

// Tile size / stage count: >= 3 stages where possible, then large tiles, preferring a
// footprint that lets two CTAs share an SM.  `align` = tile granularity (points).
bool try_pick_tiles(int nu, size_t prefix, int Tmax, int Tmin0, bool fine, TileChoice& out, bool upd = false) {
  // A bulk copy costs the TMA unit ~85 ns whatever its size (measured in the block-iteration
  // kernel), so kernels that stage many vectors per tile first try for copies of >= min_copy
  // bytes (fewer stages, one CTA per SM) before falling back to the small-tile choices.
  // Measured (A/B on one box): 2 KB copies for nu >= 16 -- C4 6.77 -> 6.97 s-steps/s (block-MGS
  // update 5.5 -> 5.8 TB/s, cross products 4.5 -> 4.7); 4 KB for nu >= 24 helps only the s = 8
  // block update of s-Omin (C5 2.55 -> 2.87 TB/s) and costs the wide Gram products.
  static const int env_copy = std::getenv("SKC_TILE_MINCOPY") ? std::atoi(std::getenv("SKC_TILE_MINCOPY")) : -1;
  const int min_copy = env_copy >= 0 ? env_copy : (upd && nu >= 24 ? 4096 : nu >= 16 ? 2048 : 0);
  for (int pass = 0; pass < 2; ++pass) {
  const int Tmin = pass == 0 ? std::max(Tmin0, min_copy / 8) : Tmin0;
  if (pass == 0 && (min_copy == 0 || Tmin > Tmax)) continue;
  for (size_t limit : {(size_t)110 * 1024, (size_t)220 * 1024}) {
    for (int ns : {3, 4, 2}) {
      for (int T2 = 2 * Tmax; T2 >= 2 * Tmin; T2 /= 2) {
        for (int T : {T2 / 2 + T2 / 4, T2 / 2}) {  // 3/4 and 1/2 of T2: 1536, 1024, .., 96, 64
          if (T > Tmax || T < Tmin || (!fine && T != T2 / 2)) continue;
          const size_t need = 64 + prefix + (size_t)ns * nu * T * 8;
          if (need <= limit) {
            out = {T, ns, need};
            return true;
          }
        }
      }
    }
  }
  }
  return false;
}

TileChoice pick_tiles(int nu, size_t prefix, int Tmax, int Tmin, bool fine = true, bool upd = false) {
  TileChoice tc;
  if (!try_pick_tiles(nu, prefix, Tmax, Tmin, fine, tc, upd))
    fail(SKC_EINVAL, "streaming kernel: too many operand vectors for shared-memory staging");
  return tc;
}

int add_unique(const double** U, int& nu, int cap, const double* p) {
  for (int v = 0; v < nu; ++v)
    if (U[v] == p) return v;
  require(nu < cap, "streaming kernel: operand list overflow");
  U[nu] = p;
  return nu++;
}

template <class K>
void allow_smem(K* kernel) {
  ensure_smem(kernel, 227 * 1024);
}

template <int NOUT, int MAXD, int PPT, bool SPLIT>
void launch_upd_t(Ctx& c, const UpdDesc& d, size_t smem, int G) {
  allow_smem(k_upd<NOUT, MAXD, PPT, SPLIT>);
  launch_k(c, k_upd<NOUT, MAXD, PPT, SPLIT>, G, THREADS, smem, d);
}

template <int NOUT, int MAXD, int PPT>
void launch_upd_s(Ctx& c, const UpdDesc& d, size_t smem, int G) {
  // the half-split form exists for the s-Omin block update shapes (2s outputs, s = 1, 2, 4, 8)
  if constexpr (NOUT == 2 || NOUT == 4 || NOUT == 8 || NOUT == 16) {
    if (d.nin0 >= 0) return launch_upd_t<NOUT, MAXD, PPT, true>(c, d, smem, G);
  }
  launch_upd_t<NOUT, MAXD, PPT, false>(c, d, smem, G);
}

template <int NOUT, int PPT>
void launch_upd_d(Ctx& c, const UpdDesc& d, size_t smem, int G, int maxd) {
  switch (maxd) {
    case 0: launch_upd_s<NOUT, 0, PPT>(c, d, smem, G); break;
    case 1: launch_upd_s<NOUT, 1, PPT>(c, d, smem, G); break;
    case 4: launch_upd_s<NOUT, 4, PPT>(c, d, smem, G); break;
    case 16: launch_upd_s<NOUT, 16, PPT>(c, d, smem, G); break;
    default: launch_upd_s<NOUT, 64, PPT>(c, d, smem, G); break;
  }
}

template <int NOUT>
void launch_upd_p(Ctx& c, const UpdDesc& d, size_t smem, int G, int maxd) {
  if (d.h.T == 2 * CONS && NOUT <= 8)
    launch_upd_d<NOUT, (NOUT <= 8 ? 2 : 1)>(c, d, smem, G, maxd);
  else
    launch_upd_d<NOUT, 1>(c, d, smem, G, maxd);
}

template <int NR, int LB>
void launch_grm_t(Ctx& c, const GrmDesc& d, size_t smem, int G) {
  allow_smem(k_grm<NR, LB>);
  launch_k(c, k_grm<NR, LB>, G, THREADS, smem, d);
}

// LB = ceil(nl / 8) rows per warp so all eight consumer warps carry a share of the rows
template <int NR>
void launch_grm_l(Ctx& c, const GrmDesc& d, size_t smem, int G) {
  switch ((d.nl + NCW - 1) / NCW) {
    case 1: launch_grm_t<NR, 1>(c, d, smem, G); break;
    case 2: launch_grm_t<NR, 2>(c, d, smem, G); break;
    case 3: launch_grm_t<NR, 3>(c, d, smem, G); break;
    case 4: launch_grm_t<NR, 4>(c, d, smem, G); break;
    case 5: launch_grm_t<NR, 5>(c, d, smem, G); break;
    case 6: launch_grm_t<NR, 6>(c, d, smem, G); break;
    case 7: launch_grm_t<NR, 7>(c, d, smem, G); break;
    default: launch_grm_t<NR, 8>(c, d, smem, G); break;
  }
}

template <int S, bool DOTS>
void launch_mgs_t(Ctx& c, const MgsDesc& d, size_t smem, int G) {
  if constexpr (DOTS && S >= 6) {
    allow_smem(k_mgs2<S>);
    launch_k(c, k_mgs2<S>, G, THREADS, smem, d);
  } else {
    allow_smem(k_mgs<S, DOTS>);
    launch_k(c, k_mgs<S, DOTS>, G, THREADS, smem, d);
  }
}

void fill_hdr(PipeHdr& h, int nu, const TileChoice& tc, int64_t n, int64_t range, int G, int cpg, int64_t gsize,
              const int* halt, const int* cond) {
  h.nu = nu;
  h.T = tc.T;
  h.nstage = tc.nstage;
  h.n = n;
  h.range = range;
  h.cpg = cpg > 0 ? cpg : G;  // (descriptors without a geometry: one group of all G CTAs)
  h.gsize = cpg > 0 ? gsize : n;
  h.halt = halt;
  h.cond = cond;
}

template <int S>
void launch_bupd_t(Ctx& c, const BupdDesc& d, size_t smem, int G, bool dots) {
  if (dots) {
    allow_smem(k_bupd<S, true>);
    launch_k(c, k_bupd<S, true>, G, THREADS, smem, d);
  } else {
    allow_smem(k_bupd<S, false>);
    launch_k(c, k_bupd<S, false>, G, THREADS, smem, d);
  }
}

// The s-Omin half-block update shape (see k_bupd): S = 5..8 unscaled outputs, whole blocks of S
// dense terms with one contiguous coefficient array, no products or exactly the upper-triangle
// Gram of the outputs followed by their products with one extra vector.  Anything else (and
// SKC_BUPD=0) takes k_upd.
bool try_launch_bupd(Ctx& c, const LinDesc& L, const char* name) {
  const int S = L.nout;
  if (!c.bupd || S < 5 || S > kMaxS || L.nin < S || L.nin % S != 0) return false;
  const bool dots = L.nd > 0;
  if (dots ? (L.nx != 1 || L.nd != S * (S + 1) / 2 + S) : L.nx != 0) return false;
  for (int q = 0; q < S; ++q)
    if (L.bscale[q] >= 0) return false;
  const unsigned all = (1u << S) - 1u;
  for (int j = 0; j < L.nin; ++j)
    if (L.mask[j] != all || L.cbase[j] != L.cbase[0] + j * S) return false;
  if (L.cbase[0] < 0 || L.cbase[0] + L.nin * S > L.ncoef) return false;
  if (dots) {
    int k = 0;
    for (int a = 0; a < S; ++a)
      for (int b = a; b < S; ++b, ++k)
        if (L.da[k] != a || L.db[k] != b) return false;
    for (int a = 0; a < S; ++a, ++k)
      if (L.da[k] != a || L.db[k] != S) return false;
  }
  BupdDesc d;
  std::memset(&d, 0, sizeof d);
  int nu = 0;
  for (int q = 0; q < S; ++q) add_unique(d.U, nu, UPD_MAXU, L.base[q]);
  for (int j = 0; j < L.nin; ++j) add_unique(d.U, nu, UPD_MAXU, L.in[j]);
  if (dots) add_unique(d.U, nu, UPD_MAXU, L.xin[0]);
  if (nu != S + L.nin + (dots ? 1 : 0)) return false;  // repeated operands: the stage slots are positional
  for (int q = 0; q < S; ++q) d.out[q] = L.out[q];
  d.nin = L.nin;
  d.cb0 = L.cbase[0];
  d.coef = L.coef;
  d.partials = L.partials;
  d.dot0 = L.dot0;
  d.G = L.G;
  const size_t prefix = 8 * ((size_t)((L.nin * S + 15) & ~15) + (dots ? (size_t)NCW * (S * (S + 1) / 2 + S) : 0));
  const size_t stage = (size_t)nu * BUPD_T * 8;
  const size_t room = (size_t)224 * 1024 - 64 - prefix;
  const int ns = (int)std::min<size_t>(kMaxStage, room / stage);
  if (ns < 2) return false;
  const TileChoice tc{BUPD_T, ns, 64 + prefix + (size_t)ns * stage};
  fill_hdr(d.h, nu, tc, L.n, L.range, L.G, L.cpg, L.gsize, L.halt, L.cond);
  const double bytes = 8.0 * (double)L.n * (nu + S);
  Launch lh(c, name, bytes);
  switch (S) {
    case 5: launch_bupd_t<5>(c, d, tc.smem, L.G, dots); break;
    case 6: launch_bupd_t<6>(c, d, tc.smem, L.G, dots); break;
    case 7: launch_bupd_t<7>(c, d, tc.smem, L.G, dots); break;
    default: launch_bupd_t<8>(c, d, tc.smem, L.G, dots); break;
  }
  CK(cudaGetLastError());
  return true;
}

template <int S>
void launch_bupd2_t(Ctx& c, const Bupd2Desc& d, size_t smem, int G) {
  allow_smem(k_bupd2<S>);
  launch_k(c, k_bupd2<S>, G, THREADS, smem, d);
}

// The fused s-Omin block update shape at s = 2..4 (see k_bupd2).
bool try_launch_bupd2(Ctx& c, const LinDesc& L, const char* name) {
  if (!c.bupd || L.nout % 2 != 0) return false;
  const int S = L.nout / 2;
  if (S < 2 || S > 4 || L.nin < 2 * S || L.nin % (2 * S) != 0) return false;
  if (L.nx != 1 || L.nd != S * (S + 1) / 2 + S) return false;
  for (int q = 0; q < 2 * S; ++q)
    if (L.bscale[q] >= 0) return false;
  const unsigned lo = (1u << S) - 1u, hi = lo << S;
  const int cb0 = L.cbase[0];
  for (int j = 0; j < L.nin; ++j) {
    const int e = j / (2 * S), r = j % (2 * S);
    const bool ap = r >= S;
    const int l = ap ? r - S : r;
    if (L.mask[j] != (ap ? hi : lo) || L.cbase[j] != cb0 + (e * S + l) * S - (ap ? S : 0)) return false;
  }
  if (cb0 < 0 || cb0 + (L.nin / 2) * S > L.ncoef) return false;
  {
    int k = 0;
    for (int a = 0; a < S; ++a)
      for (int b = a; b < S; ++b, ++k)
        if (L.da[k] != S + a || L.db[k] != S + b) return false;
    for (int a = 0; a < S; ++a, ++k)
      if (L.da[k] != S + a || L.db[k] != 2 * S) return false;
  }
  Bupd2Desc d;
  std::memset(&d, 0, sizeof d);
  int nu = 0;
  for (int q = 0; q < 2 * S; ++q) {
    d.ub[q] = (uint8_t)add_unique(d.U, nu, UPD_MAXU, L.base[q]);
    d.out[q] = L.out[q];
  }
  d.nb0 = nu;
  for (int j = 0; j < L.nin; ++j) add_unique(d.U, nu, UPD_MAXU, L.in[j]);
  if (nu != d.nb0 + L.nin) return false;  // repeated operands: the term slots are positional
  d.ix = add_unique(d.U, nu, UPD_MAXU, L.xin[0]);
  d.nin = L.nin;
  d.cb0 = cb0;
  d.coef = L.coef;
  d.partials = L.partials;
  d.dot0 = L.dot0;
  d.G = L.G;
  const size_t prefix = 8 * ((size_t)(((L.nin / 2) * S + 15) & ~15) + (size_t)NCW * (S * (S + 1) / 2 + S));
  const size_t stage = (size_t)nu * BUPD_T * 8;
  const size_t room = (size_t)224 * 1024 - 64 - prefix;
  const int ns = (int)std::min<size_t>(kMaxStage, room / stage);
  if (ns < 2) return false;
  const TileChoice tc{BUPD_T, ns, 64 + prefix + (size_t)ns * stage};
  fill_hdr(d.h, nu, tc, L.n, L.range, L.G, L.cpg, L.gsize, L.halt, L.cond);
  const double bytes = 8.0 * (double)L.n * (nu + 2 * S);
  Launch lh(c, name, bytes);
  switch (S) {
    case 2: launch_bupd2_t<2>(c, d, tc.smem, L.G); break;
    case 3: launch_bupd2_t<3>(c, d, tc.smem, L.G); break;
    default: launch_bupd2_t<4>(c, d, tc.smem, L.G); break;
  }
  CK(cudaGetLastError());
  return true;
}

}  // namespace

void launch_lincomb(Ctx& c, const LinDesc& L, const char* name) {
  require(L.nin <= LC_MAXIN && L.nout <= LC_MAXOUT && L.nx <= LC_MAXX && L.nd <= LC_MAXD,
          "lincomb: descriptor too large");
  require(L.nout >= 1, "lincomb: no outputs");
  if (try_launch_bupd(c, L, name) || try_launch_bupd2(c, L, name)) return;
  static const int kOut[] = {1, 2, 3, 4, 7, 8, 16};
  int nout_t = 16;
  for (int v : kOut)
    if (v >= L.nout) {
      nout_t = v;
      break;
    }
  UpdDesc d;
  std::memset(&d, 0, sizeof d);
  int nu = 0;
  d.nin = L.nin;
  d.nout = nout_t;
  d.nx = L.nx;
  d.nd = L.nd;
  d.ncoef = L.ncoef;
  for (int q = 0; q < L.nout; ++q) {
    d.ub[q] = (uint8_t)add_unique(d.U, nu, UPD_MAXU, L.base[q]);
    d.bscale[q] = L.bscale[q];
    d.out[q] = L.out[q];
  }
  if (nout_t != L.nout) {  // padded outputs: copies of output 0's base into a scratch vector
    double* pad = (double*)c.workspace("lincomb_pad", (size_t)(L.n + 32) * sizeof(double));
    for (int q = L.nout; q < nout_t; ++q) {
      d.ub[q] = d.ub[0];
      d.bscale[q] = -1;
      d.out[q] = pad;
    }
  }
  // half-split shape: every term feeds exactly the first or the second half of the outputs
  // (s-Omin's P / AP block update).  Terms are then ordered low half first, each half in its
  // original order -- the per-output accumulation order is unchanged.
  d.nin0 = -1;
  if (nout_t == L.nout && L.nout % 2 == 0 && L.nout >= 2) {
    const unsigned lo = (1u << (L.nout / 2)) - 1u, hi = lo << (L.nout / 2);
    bool split = true;
    for (int j = 0; j < L.nin && split; ++j) split = L.mask[j] == lo || L.mask[j] == hi;
    if (split) {
      int w = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < L.nin; ++j)
          if ((L.mask[j] == lo) == (pass == 0)) {
            d.ut[w] = (uint8_t)add_unique(d.U, nu, UPD_MAXU, L.in[j]);
            d.mask[w] = L.mask[j];
            d.cbase[w] = L.cbase[j];
            ++w;
          }
      d.nin0 = 0;
      for (int j = 0; j < L.nin; ++j) d.nin0 += L.mask[j] == lo;
    }
  }
  if (d.nin0 < 0) {
    for (int j = 0; j < L.nin; ++j) {
      d.ut[j] = (uint8_t)add_unique(d.U, nu, UPD_MAXU, L.in[j]);
      d.mask[j] = L.mask[j];
      d.cbase[j] = L.cbase[j];
    }
  }
  for (int x = 0; x < L.nx; ++x) d.ux[x] = (uint8_t)add_unique(d.U, nu, UPD_MAXU, L.xin[x]);
  for (int k = 0; k < L.nd; ++k) {  // value ids: outputs, then extras at NOUT + x
    d.da[k] = (uint8_t)(L.da[k] < L.nout ? L.da[k] : L.da[k] - L.nout + nout_t);
    d.db[k] = (uint8_t)(L.db[k] < L.nout ? L.db[k] : L.db[k] - L.nout + nout_t);
  }
  const int maxd = L.nd == 0 ? 0 : L.nd <= 1 ? 1 : L.nd <= 4 ? 4 : L.nd <= 16 ? 16 : 64;
  d.coef = L.coef;
  d.partials = L.partials;
  d.dot0 = L.dot0;
  d.G = L.G;
  const size_t prefix = 8 * ((size_t)((L.ncoef + 15) & ~15) + (maxd ? (size_t)(nout_t + L.nx) * CONS : 0));
  // k_upd covers T <= CONS * PPT points per tile (powers of two only).  A tile of at least CONS
  // points keeps every consumer thread busy (one point each) -- worth one CTA per SM with
  // fewer stages for wide updates (the seed and x updates stream up to 4 + m s vectors).
  TileChoice tc;
  const int Tmax = nout_t <= 8 ? 2 * CONS : CONS;
  if (!try_pick_tiles(nu, prefix, Tmax, CONS, false, tc, true)) tc = pick_tiles(nu, prefix, Tmax, 64, false, true);
  fill_hdr(d.h, nu, tc, L.n, L.range, L.G, L.cpg, L.gsize, L.halt, L.cond);
  const double bytes = 8.0 * (double)L.n * (nu + L.nout);
  Launch lh(c, name, bytes);
  switch (nout_t) {
    case 1: launch_upd_p<1>(c, d, tc.smem, L.G, maxd); break;
    case 2: launch_upd_p<2>(c, d, tc.smem, L.G, maxd); break;
    case 3: launch_upd_p<3>(c, d, tc.smem, L.G, maxd); break;
    case 4: launch_upd_p<4>(c, d, tc.smem, L.G, maxd); break;
    case 7: launch_upd_p<7>(c, d, tc.smem, L.G, maxd); break;
    case 8: launch_upd_p<8>(c, d, tc.smem, L.G, maxd); break;
    default: launch_upd_p<16>(c, d, tc.smem, L.G, maxd); break;
  }
  CK(cudaGetLastError());
}

void launch_gram(Ctx& c, const GramDesc& g, const char* name) {
  require(g.nl >= 1 && g.nl <= GR_MAXL && g.nr >= 1 && g.nr <= GR_MAXR, "gram: descriptor out of range");
  GrmDesc d;
  std::memset(&d, 0, sizeof d);
  int nu = 0;
  d.nl = g.nl;
  d.nr = g.nr;
  for (int l = 0; l < g.nl; ++l) d.li[l] = (uint8_t)add_unique(d.U, nu, GRM_MAXU, g.L[l]);
  for (int r = 0; r < g.nr; ++r) {
    d.ri[r] = (uint8_t)add_unique(d.U, nu, GRM_MAXU, g.R[r]);
    d.rbase[r] = g.mapped ? g.rbase[r] : g.dot0 + r;
    d.rstride[r] = g.mapped ? g.rstride[r] : g.nr;
    d.lmax[r] = g.mapped ? g.lmax[r] : g.nl;
  }
  d.partials = g.partials;
  d.G = g.G;
  TileChoice tc = pick_tiles(nu, 0, 2048, 64);
  const size_t red = 64 + (size_t)NCW * 8 * GR_MAXR * 8;
  tc.smem = std::max(tc.smem, red);
  fill_hdr(d.h, nu, tc, g.n, g.range, g.G, g.cpg, g.gsize, g.halt, g.cond);
  const double bytes = 8.0 * (double)g.n * nu;
  Launch lh(c, name, bytes);
  switch (g.nr) {
    case 1: launch_grm_l<1>(c, d, tc.smem, g.G); break;
    case 2: launch_grm_l<2>(c, d, tc.smem, g.G); break;
    case 3: launch_grm_l<3>(c, d, tc.smem, g.G); break;
    case 4: launch_grm_l<4>(c, d, tc.smem, g.G); break;
    case 5: launch_grm_l<5>(c, d, tc.smem, g.G); break;
    case 6: launch_grm_l<6>(c, d, tc.smem, g.G); break;
    case 7: launch_grm_l<7>(c, d, tc.smem, g.G); break;
    default: launch_grm_l<8>(c, d, tc.smem, g.G); break;
  }
  CK(cudaGetLastError());
}

void launch_mgs(Ctx& c, const Geo& geo, int s, const double* const* Vi, double* const* cand, const double* const* Vnext,
                const MgsScalar& sc, double* partials, int dot0, const int* halt, const int* cond,
                const char* name) {
  require(s >= 2 && s <= kMaxS, "mgs: s out of range");
  MgsDesc d;
  std::memset(&d, 0, sizeof d);
  int nu = 0;
  for (int l = 0; l < s; ++l) d.U[nu++] = Vi[l];
  for (int j = 1; j < s; ++j) {
    d.U[nu++] = cand[j];
    d.cand[j - 1] = cand[j];
  }
  const bool dots = Vnext != nullptr;
  if (dots)
    for (int l = 0; l < s; ++l) d.U[nu++] = Vnext[l];
  d.sc = sc;
  d.partials = partials;
  d.dot0 = dot0;
  d.G = geo.G;
  TileChoice tc = pick_tiles(nu, kMgsPrefix, 2048, 64);
  tc.smem = std::max(tc.smem, 64 + (size_t)kMgsPrefix + 8 * (size_t)NCW * 56);
  fill_hdr(d.h, nu, tc, geo.n, geo.range, geo.G, geo.cpg, geo.gsize, halt, cond);
  const double bytes = 8.0 * (double)geo.n * (nu + s - 1);
  Launch lh(c, name, bytes);
#define SKC_MGS_CASE(SV)                                                \
  case SV:                                                              \
    if (dots)                                                           \
      launch_mgs_t<SV, true>(c, d, tc.smem, geo.G);                     \
    else                                                                \
      launch_mgs_t<SV, false>(c, d, tc.smem, geo.G);                    \
    break;
  switch (s) {
    SKC_MGS_CASE(2)
    SKC_MGS_CASE(3)
    SKC_MGS_CASE(4)
    SKC_MGS_CASE(5)
    SKC_MGS_CASE(6)
    SKC_MGS_CASE(7)
    SKC_MGS_CASE(8)
  }
#undef SKC_MGS_CASE
  CK(cudaGetLastError());
}

}  // namespace skc
