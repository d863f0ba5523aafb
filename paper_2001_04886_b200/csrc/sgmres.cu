// sgmres.cu -- device-resident s-step Arnoldi (sstep.hpp:271-458), s-step GMRES(m)
// (sstep.hpp:493-654), sarnoldi (sstep.hpp:465-485) and the standard MGS-GMRES(m) used for
// s = 1 and as the basis-collapse fallback (solvers.hpp:86-110, 297-359).
//
// One restart cycle (constructor + m block iterations, every Scalar1/Scalar2 Gram solve,
// block-MGS pass, reorthogonalization test and basis push, and the least-squares half: the
// block-Hessenberg columns (append_g_columns), cholesky_upper of each Gram block, the Givens
// update with the early exit rho <= tol, the back substitution, x += V y and r = f - A x) is
// enqueued without a host round trip, as one CUDA graph.  The s x s solves and every decision
// run on the device (lsq.cuh, small_dense.cuh); the host synchronizes once per cycle and
// replays the reference's control flow on the device's records to build the SolveReport
// (history, op counts, breakdown strings) -- it computes no numbers of its own.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "device_util.cuh"
#include "lsq.cuh"
#include "solver_util.hpp"
#include "stencil.cuh"

namespace skc {

namespace {

// cycle status: running, or what stopped it (and at which block, ArnState::block)
enum : int {
  kArnRunning = 0,
  kArnCtorZero = 1,       // start vector zero (the reference's require, sstep.hpp:277)
  kArnCtorCollapse = 2,   // push_block of block 0 (basis collapse at the constructor)
  kArnInvariant = 3,      // nu <= 1e-14 ||z|| (sstep.hpp:320-324)
  kArnPushCollapse = 4,   // push_block of block k (sstep.hpp:375)
  kArnCholCollapse = 5,   // cholesky_upper of block k's Gram matrix (sstep.hpp:585)
  kArnCtorChol = 6,       // cholesky_upper of block 0 (escapes sgmres_solve, sstep.hpp:563)
  kArnEarly = 7,          // rho <= tol after block k (sstep.hpp:600)
};
// end-of-cycle outcome (k_arn_finish)
enum : int { kFinNone = 0, kFinOk = 1, kFinFallback = 2, kFinLsqFail = 3 };

struct ArnState {
  int status;
  int halt;
  int block;   // block iteration that stopped the cycle
  int reorth;  // reorthogonalization flag of the current block iteration
  double rn;   // latest residual norm (also the constructor's ||r||)
  int zready;  // the last block iteration's cross pass produced the next z and its products
  int fixed;   // fixed-step benchmark mode (gram_bypass_ratio, lsq_solve)
  int fin;     // end-of-cycle outcome (kFin*)
  // the least-squares stream's verdict on the block steps (kArnRunning, kArnInvariant,
  // kArnPushCollapse, kArnCholCollapse, kArnEarly) and its step; written only by
  // k_arn_lsq, which also raises the sticky `halt` so later block steps return at entry
  int lstatus, lblock;
  // block-iteration kernel: the halt flag as CTA 0 read it (the whole grid's decision after the
  // first grid barrier) and the monotonic arrival counter of its grid barriers
  int hseen;
  alignas(128) unsigned long long gbar;  // (a cache line of its own: the flags above are polled by other kernels)
};

// record layout per block iteration k (0 = constructor)
// (W: the pushed Gram matrix as symmetrized by push_block; Wraw: the candidate's raw products,
// snapshotted at the end of its block step for the least-squares stream)
struct RecLayout {
  int s, m;
  __host__ __device__ int size() const { return 10 + 2 * s * s + (m + 1) * s + (m + 1) * s * s; }
  static constexpr int kZn = 0, kNu = 1, kInv = 2, kReorth = 3, kFirst = 4, kOk = 5, kRatio = 6, kSing = 7,
                       kRho = 8, kW = 10;
  __host__ __device__ int wraw() const { return 10 + s * s; }
  __host__ __device__ int h() const { return 10 + 2 * s * s; }
  __host__ __device__ int t() const { return 10 + 2 * s * s + (m + 1) * s; }
};

// coefficient layout
struct CoefLayout {
  int s, m;
  int H() const { return 0; }
  int T() const { return m * s; }
  int Inv() const { return m * s + s * s; }
  int Y() const { return Inv() + 1; }
  int M1() const { return Y() + (m + 1) * s; }
  int size() const { return M1() + 1; }
};

// dot-region layout
struct DotLayout {
  int s, m;
  int Z() const { return 0; }
  int Seed() const { return m * s + 1; }
  int D() const { return Seed() + 1; }
  // block-MGS products, double-buffered by round: round i reads Dr(i) and writes Dr(i+1)
  int Dr(int i) const { return D() + (i & 1) * s * s; }
  int Cross() const { return D() + 2 * s * s; }
  int Wa() const { return Cross() + m * s * s; }
  int Wb() const { return Wa() + s * s; }
  int RR() const { return Wb() + s * s; }
  int size() const { return RR() + 1; }
};

__device__ __forceinline__ bool arn_skip(const ArnState* st) { return st->halt != 0; }

// SStepArnoldi ctor scale (sstep.hpp:276-279). use_rn: reuse the residual norm computed by
// checked_norm (same vector, same reduction => same value as the reference's norm2(v1)).
__global__ void k_arn_ctor(ArnState* st, int use_rn, const double* partials, int G, int dNV, double* rec0,
                           double* coef, int cInv) {
  SKC_PDL_ENTRY();
  __shared__ double v[1];
  if (!use_rn) reduce_dots_dev(partials, G, dNV, 1, v);
  if (threadIdx.x == 0) {
    st->status = kArnRunning;
    st->halt = 0;
    st->block = 0;
    st->reorth = 0;
    st->zready = 0;
    st->fin = kFinNone;
    st->lstatus = kArnRunning;
    st->lblock = 0;
    const double nv = use_rn ? st->rn : sqrt(v[0]);
    rec0[RecLayout::kZn] = nv;
    if (!(nv > 0.0)) {
      st->status = kArnCtorZero;
      st->halt = 1;
      return;
    }
    coef[cInv] = 1.0 / nv;
  }
}

// push_block (sstep.hpp:392-399): W = gram_self(block) -> GramSolver; breakdown = collapse.
// One thread, on the reduced s x s products v; the factor is built in g (scratch) and stored
// to grams[k] by the caller when the status stays running.  S > 0: compile-time order.
template <int S = 0>
__device__ bool arn_push_body(ArnState* st, Gram& g, int k, double* rec, const double* v, int s, bool record = true) {
  double W[kMaxS * kMaxS];
  if constexpr (S > 0) {
#pragma unroll
    for (int q = 0; q < S * S; ++q) W[q] = v[q];
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int l = j + 1; l < S; ++l) {
        const double avg = (W[j * S + l] + W[l * S + j]) / 2.0;
        W[j * S + l] = avg;
        W[l * S + j] = avg;
      }
    gram_factor_t<S>(g, W);
  } else {
    for (int q = 0; q < s * s; ++q) W[q] = v[q];
    for (int j = 0; j < s; ++j)
      for (int l = j + 1; l < s; ++l) {
        const double avg = (W[j * s + l] + W[l * s + j]) / 2.0;
        W[j * s + l] = avg;
        W[l * s + j] = avg;
      }
    gram_factor_dev(g, W, s);
  }
  gram_bypass_ratio(g, st->fixed);
  if (!record) return g.ok;
  if constexpr (S > 0) {
#pragma unroll
    for (int q = 0; q < S * S; ++q) rec[RecLayout::kW + q] = W[q];
  } else {
    for (int q = 0; q < s * s; ++q) rec[RecLayout::kW + q] = W[q];
  }
  rec[RecLayout::kOk] = g.ok;
  rec[RecLayout::kRatio] = g.ratio;
  rec[RecLayout::kSing] = g.singular1;
  if (!g.ok) {
    st->status = k == 0 ? kArnCtorCollapse : kArnPushCollapse;
    st->block = k;
    st->halt = 1;
    return false;
  }
  return true;
}

// per-round path: push_block of block k from the reduced W products (the reorthogonalized region
// when the flag says so); the raw products are kept in the record for the least-squares stream
__global__ void k_arn_push(ArnState* st, Gram* grams, int k, double* rec, int rec_wraw, const double* partials, int G,
                           int dWa, int dWb, int s) {
  SKC_PDL_ENTRY();
  if (arn_skip(st)) return;
  __shared__ double v[kMaxS * kMaxS];
  const int dW = st->reorth ? dWb : dWa;
  reduce_dots_dev(partials, G, dW, s * s, v);
  if (threadIdx.x == 0) {
    for (int q = 0; q < s * s; ++q) rec[rec_wraw + q] = v[q];
    Gram g;
    if (arn_push_body(st, g, k, rec, v, s)) grams[k] = g;
  }
}

// ---------------------------------------------------------------- least squares of the cycle
// Device state of sgmres_solve's cycle loop (sstep.hpp:560-600): the block Hessenberg columns,
// the L blocks and the Givens least squares (lsq.cuh), written by one CTA after each block step.
struct ArnLsqDesc {
  int s, m;
  int GL;            // row stride of gcols (m s + 2)
  int lsq_on;        // 0: sarnoldi (Hessenberg columns only, no L / Givens)
  double tol;        // cfg.tol (absolute)
  double* gcols;     // block Hessenberg column j (rows 0..j+1) at j * GL, unscaled
  double* lblk;      // upper Cholesky factor of basis block b's Gram matrix at b s^2
  void* lsq;         // LsqView base, capacity m s
  double* rec;       // records (RecLayout), block iteration k at k * recsz
  int recsz, rec_t, rec_h, rec_wraw;
  ArnState* st;
  Gram* grams;
  unsigned long long* trace;  // optional per-phase timestamps (slots 70..75), diagnostics
};
__device__ __forceinline__ void lsq_mark(const ArnLsqDesc& d, int slot, int who = 0) {
  if (d.trace && threadIdx.x == who) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    d.trace[slot] = t;
  }
}
__host__ __device__ inline int arn_lsq_ld(int s, int m) { return m * s + 2; }
// shared scratch of arn_lsq_step (doubles) without / with the staged earlier Hessenberg columns
__host__ __device__ inline int arn_lsq_scratch(int s, int m) {
  const int M = m * s;
  return 3 * s * arn_lsq_ld(s, m) + (m * s * s) + (M + 1) + (m + 1) * s * s + 2 * (M + s) + 16;
}
__host__ __device__ inline int arn_lsq_prev(int s, int m) {
  const int M = m * s;
  return M * (M + 3) / 2;
}

// Block step k's half of the cycle loop (sstep.hpp:582-600), one whole CTA, on the side stream
// once block step k has finished (the next block step runs meanwhile):
//   the push_block decision for the candidate (sstep.hpp:375, 392-399; when it was built: k < m
//   and the seed did not vanish), recomputed from the snapshotted raw Gram products with the
//   same arithmetic as the block step kernels' own push (hence the same verdict), then
//   cholesky_upper of the new Gram block (sstep.hpp:585); either failing is a basis collapse
//   and appends nothing;
//   append_g_columns (sstep.hpp:422-445): the s columns of step k from the t coefficients of
//   block k-1 and this step's h, nu;
//   apply_l (sstep.hpp:566-579) and the Givens update of each column (lsq.cuh); rho is recorded
//   and rho <= tol stops the cycle.
// Every stop raises the sticky st->halt, so the block steps not yet started return at entry
// (the one running meanwhile finishes; nothing reads its results).  Latency-bound serial work:
// every operand is staged into shared memory in one parallel pass, computed there, and
// written back without waiting.  `cap` = doubles of scratch available.
template <int S>
__device__ void arn_lsq_step(const ArnLsqDesc& d, int k, bool build_next, double* sm, int cap) {
  __shared__ int s_go, s_nl, s_inv;
  __shared__ double s_w[S * S];
  const int tid = threadIdx.x, nt = blockDim.x;
  double* rk = d.rec + (size_t)k * d.recsz;
  const int q = k - 1, ld = arn_lsq_ld(S, d.m), j0 = q * S;
  // scratch: gs | ls | cp [S ld each] | tq [q S^2] | hk [k S + 1] | lb [(k+1) S^2] | cs, sn [j0 + S] | prev
  double* gs = sm;
  double* ls = gs + S * ld;
  double* cp = ls + S * ld;
  double* tq = cp + S * ld;
  double* hk = tq + q * S * S;
  double* lb = hk + k * S + 1;
  double* ccs = lb + (k + 1) * S * S;
  double* csn = ccs + j0 + S;
  double* prev = csn + j0 + S;
  const int nprev = j0 * (j0 + 3) / 2;  // columns 0..j0-1, column p rows 0..p+1 at p(p+3)/2
  const bool stage_prev = (int)(prev - sm) + nprev <= cap;
  const LsqView lv = lsq_view(d.lsq, d.m * S);
  lsq_mark(d, 70);
  if (tid == 0) {
    const bool invariant = rk[RecLayout::kInv] != 0.0;
    s_inv = invariant;
    int go = d.st->lstatus == kArnRunning, nl = k;
    if (go && build_next && !invariant) {
#pragma unroll
      for (int e = 0; e < S * S; ++e) s_w[e] = rk[d.rec_wraw + e];
      Gram g;
      if (!arn_push_body<S>(d.st, g, k, rk, s_w, S, false)) {
        d.st->lstatus = kArnPushCollapse;
        d.st->lblock = k;
        d.st->halt = 1;
        go = 0;
      } else if (d.lsq_on) {
        if (!cholesky_upper(g.w, S, lb + k * S * S)) {
          d.st->lstatus = kArnCholCollapse;
          d.st->lblock = k;
          d.st->halt = 1;
          go = 0;
        }
        nl = k + 1;
      }
    }
    s_go = go;
    s_nl = nl;
    lsq_mark(d, 76);
  } else {
    // stage the operands (threads 1..): t of block q, h and nu of step k, L blocks 0..k-1,
    // the stored rotations, the earlier Hessenberg columns -- one combined index space, eight
    // loads in flight per thread before their shared-memory stores
    const double* rq = d.rec + (size_t)q * d.recsz + d.rec_t;
    const int t1 = tid - 1, n1 = nt - 1;
    const int n_t = q * S * S, n_h = k * S + 1, n_l = d.lsq_on ? k * S * S : 0, n_c = d.lsq_on ? j0 : 0;
    const int n_p = stage_prev ? nprev : 0;
    const int o_h = n_t, o_l = o_h + n_h, o_c = o_l + n_l, o_s = o_c + n_c, o_p = o_s + n_c, T = o_p + n_p;
    auto src = [&](int e) -> const double* {
      if (e < o_h) return rq + e;
      if (e < o_l) return e - o_h < k * S ? rk + d.rec_h + (e - o_h) : rk + RecLayout::kNu;
      if (e < o_c) return d.lblk + (e - o_l);
      if (e < o_s) return lv.cs + (e - o_c);
      if (e < o_p) return lv.sn + (e - o_s);
      const int f = e - o_p;  // -> (column p, row r), p(p+3)/2 <= f
      int p = (int)((sqrtf(9.0f + 8.0f * (float)f) - 3.0f) * 0.5f);
      while ((p + 1) * (p + 4) / 2 <= f) ++p;
      while (p * (p + 3) / 2 > f) --p;
      return d.gcols + (size_t)p * d.GL + (f - p * (p + 3) / 2);
    };
    auto dst = [&](int e) -> double* {
      if (e < o_h) return tq + e;
      if (e < o_l) return hk + (e - o_h);
      if (e < o_c) return lb + (e - o_l);
      if (e < o_s) return ccs + (e - o_c);
      if (e < o_p) return csn + (e - o_s);
      return prev + (e - o_p);
    };
    constexpr int U = 8;
    for (int b = t1; b < T; b += U * n1) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = b + u * n1;
        v[u] = e < T ? __ldcg(src(e)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = b + u * n1;
        if (e < T) *dst(e) = v[u];
      }
    }
    lsq_mark(d, 77, 1);
  }
  __syncthreads();
  lsq_mark(d, 71);
  if (!s_go) return;
  if (build_next && !s_inv && d.lsq_on)  // the new L block to global memory
    for (int e = tid; e < S * S; e += nt) d.lblk[k * S * S + e] = lb[k * S * S + e];
  const bool invariant = s_inv != 0;
  const int nl = s_nl;
  auto prevv = [&](int p, int r) {
    return stage_prev ? prev[p * (p + 3) / 2 + r] : d.gcols[(size_t)p * d.GL + r];
  };
  // ---- append_g_columns: the s columns of step k (column j = j0 + cl, rows 0..j+1)
  for (int e = tid; e < S * ld; e += nt) {
    const int cl = e / ld, r = e - cl * ld;
    const int j = j0 + cl;
    if (r >= j + 2) continue;
    double v;
    if (cl + 1 < S) {  // A v_q^cl = v_q^{cl+1} + sum_i V_i T_i[:,cl+1] - sum_i (A V_i) T_i[:,cl]
      v = 0.0;
      if (r == j0 + cl + 1) v += 1.0;
      for (int i = 0; i < q; ++i) {
        const double* ti = tq + i * S * S;
        if (r >= i * S && r < i * S + S) v += ti[(r - i * S) * S + cl + 1];
#pragma unroll
        for (int lc = 0; lc < S; ++lc) {
          const double cf = ti[lc * S + cl];
          if (cf == 0.0) continue;
          const int pj = i * S + lc;  // earlier column, rows 0..pj+1
          if (r < pj + 2) v -= cf * prevv(pj, r);
        }
      }
    } else {  // A v_q^{s-1} = nu v_{q+1} + sum_i V_i h_i
      v = hk[r];
    }
    gs[e] = v;
    d.gcols[(size_t)j * d.GL + r] = v;
  }
  if (!d.lsq_on) {
    __syncthreads();
    return;
  }
  __syncthreads();
  lsq_mark(d, 72);
  // ---- apply_l: the L-scaled columns (and a copy for the squared norms)
  for (int e = tid; e < S * ld; e += nt) {
    const int cl = e / ld, r = e - cl * ld;
    const int len = j0 + cl + 2;
    if (r >= len) continue;
    const double* g = gs + cl * ld;
    const int bi = r / S, off = bi * S, rl = r - off;
    double v = g[r];
    if (bi < nl) {
      const double* lbb = lb + bi * S * S;
      double acc = 0.0;
      for (int jl = rl; jl < S && off + jl < len; ++jl) acc += lbb[rl * S + jl] * g[off + jl];
      v = acc;
    }
    ls[e] = v;
    cp[e] = v;
  }
  __syncthreads();
  lsq_mark(d, 73);
  // ---- Givens (HessenbergLsq::append_column per column): squared norms on thread 0 from the
  //      copy; warp 1 rotates -- lane c column c through the stored pairs, then lane 0 the pairs
  //      made inside this step and each column's new rotation
  __shared__ double s_res;
  if (tid == 0) {
    double g = lv.h->gnorm_sq;
    for (int c = 0; c < S; ++c)
      for (int i = 0; i < j0 + c + 2; ++i) g += cp[c * ld + i] * cp[c * ld + i];
    lv.h->gnorm_sq = g;
  } else if (tid >= 32 && tid < 64) {
    const int c = tid - 32;
    if (c < S) {
      double* col = ls + c * ld;
      double a = col[0];
      for (int t = 0; t < j0; ++t) {
        const double b = col[t + 1], cc = ccs[t], ss = csn[t];
        col[t] = cc * a + ss * b;
        a = -ss * a + cc * b;
      }
      col[j0] = a;
    }
    __syncwarp();
    if (c == 0) {
      double rj = lv.rhs[j0];
      for (int c2 = 0; c2 < S; ++c2) {
        double* col = ls + c2 * ld;
        const int j = j0 + c2;
        for (int t = j0; t < j; ++t) {
          const double a = col[t], b = col[t + 1], cc = ccs[t], ss = csn[t];
          col[t] = cc * a + ss * b;
          col[t + 1] = -ss * a + cc * b;
        }
        const double a = col[j], b = col[j + 1];
        const double r = sd_hypot(a, b);
        double cc = 1.0, ss = 0.0;
        if (r != 0.0) {
          cc = a / r;
          ss = b / r;
        }
        ccs[j] = cc;
        csn[j] = ss;
        col[j] = r;
        const double ra = rj, rb = 0.0;
        const double nj = cc * ra + ss * rb;
        rj = -ss * ra + cc * rb;
        lv.rhs[j] = nj;
        lv.cs[j] = cc;
        lv.sn[j] = ss;
      }
      lv.rhs[j0 + S] = rj;
      s_res = sd_abs(rj);
    }
  }
  __syncthreads();
  lsq_mark(d, 74);
  // ---- write back R's new columns; header; record rho; early exit
  for (int e = tid; e < S * ld; e += nt) {
    const int cl = e / ld, r = e - cl * ld;
    const int j = j0 + cl;
    if (r <= j) lsq_r(lv, j, r) = ls[e];
  }
  lsq_mark(d, 78);
  if (tid == 0) {
    const double rho = s_res;
    lv.h->cols = j0 + S;
    lv.h->residual = rho;
    rk[RecLayout::kRho] = rho;
    if (invariant) {  // (the block step already stopped the cycle; the verdict for the host)
      d.st->lstatus = kArnInvariant;
      d.st->lblock = k;
    } else if (build_next && rho <= d.tol) {
      d.st->lstatus = kArnEarly;
      d.st->lblock = k;
      d.st->halt = 1;
    }
  }
  __syncthreads();
  lsq_mark(d, 75);
}

// the constructor's push_block of block 0, then L_0 = cholesky_upper(W_0) and
// HessenbergLsq(rn L_0(0,0)) (sstep.hpp:562-564)
template <int S>
__global__ void k_arn_ctor_push(const ArnLsqDesc d, const double* partials, int G, int dW) {
  SKC_PDL_ENTRY();
  if (d.st->halt) return;
  __shared__ double v[kMaxS * kMaxS];
  __shared__ Gram s_g0;
  reduce_dots_dev(partials, G, dW, S * S, v);
  if (threadIdx.x == 0) {
    Gram& g = s_g0;
    if (!arn_push_body<S>(d.st, g, 0, d.rec, v, S)) return;
    d.grams[0] = g;
    if (!d.lsq_on) return;
    double L[S * S];
    if (!cholesky_upper(g.w, S, L)) {
      d.st->status = kArnCtorChol;
      d.st->halt = 1;
      return;
    }
    for (int q = 0; q < S * S; ++q) d.lblk[q] = L[q];
    lsq_reset(lsq_view(d.lsq, d.m * S), d.st->rn * L[0]);
  }
}

// block step k's least squares (arn_lsq_step), on the side stream
template <int S>
__global__ void k_arn_lsq(const ArnLsqDesc d, int k, int build_next, int cap) {
  extern __shared__ __align__(16) double lsq_sm[];
  if (d.st->lstatus != kArnRunning) return;  // (an earlier step stopped the cycle)
  arn_lsq_step<S>(d, k, build_next != 0, lsq_sm, cap);
}

// end of the cycle (sstep.hpp:602-625): unless the constructor failed, a collapse with the
// residual estimate above tol hands the cycle to the fallback (x untouched); otherwise y from the
// back substitution (its rank failure is the reference's breakdown) -- y lands in the update
// coefficients, zero beyond the appended columns, so the fixed x update adds exact zeros there
// (the back substitution is a serial chain of M(M+1)/2 dependent steps: R, the right-hand side
// and y are staged in shared memory when they fit -- M <= kFinSmemCols -- else read in place)
constexpr int kFinSmemCols = 128;
__host__ __device__ inline size_t fin_smem_doubles(int M) {
  return M <= kFinSmemCols ? (size_t)M * (M + 1) / 2 + 2 * (size_t)M + 8 : 8;
}
__global__ void k_arn_finish(const ArnLsqDesc d, double* ycoef) {
  SKC_PDL_ENTRY();
  extern __shared__ __align__(16) double fin_sm[];
  __shared__ int s_go;
  const int M = d.m * d.s;
  const LsqView lv = lsq_view(d.lsq, M);
  ArnState* st = d.st;
  if (threadIdx.x == 0) {
    const int stv = st->status;
    int go = 1;
    if (stv == kArnCtorZero || stv == kArnCtorCollapse || stv == kArnCtorChol) {
      st->fin = kFinNone;
      go = 0;
    } else {
      const int ls = st->lstatus;
      const bool collapsed = ls == kArnPushCollapse || ls == kArnCholCollapse;
      const bool attainable = lv.h->cols > 0 && lv.h->residual <= d.tol;
      if (collapsed && !attainable) {
        st->fin = kFinFallback;
        go = 0;
      }
    }
    s_go = go;
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x) ycoef[i] = 0.0;
  __syncthreads();
  if (!s_go) return;
  const int cols = lv.h->cols;
  LsqHdr* sh = reinterpret_cast<LsqHdr*>(fin_sm);
  LsqView sv = lv;
  if (M <= kFinSmemCols) {  // stage R, rhs
    double* p = fin_sm + 4;
    sv.h = sh;
    sv.R = p;
    sv.rhs = p + (size_t)M * (M + 1) / 2;
    sv.y = sv.rhs + M;
    const int nr = cols * (cols + 1) / 2;
    for (int e = threadIdx.x; e < nr; e += blockDim.x) sv.R[e] = lv.R[e];
    for (int e = threadIdx.x; e < cols; e += blockDim.x) sv.rhs[e] = lv.rhs[e];
    if (threadIdx.x == 0) *sh = *lv.h;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const bool ok = lsq_solve(sv, st->fixed != 0);
    lv.h->rank_col = sv.h->rank_col;
    st->fin = ok ? kFinOk : kFinLsqFail;
    if (ok)
      for (int i = 0; i < cols; ++i) ycoef[i] = sv.y[i];
  }
}

// Scalar1 (sstep.hpp:301-310): zn = ||z||, h_i = W_i^{-1} V_i^T z
__global__ void k_arn_s1(ArnState* st, const Gram* grams, int k, double* rec, double* coef, const double* partials,
                         int G, int dZ, int s, int cH, double* scratch) {
  SKC_PDL_ENTRY();
  if (arn_skip(st)) return;
  reduce_dots_dev(partials, G, dZ, k * s + 1, scratch);
  if (threadIdx.x == 0) {
    rec[RecLayout::kZn] = sqrt(scratch[k * s]);
    rec[RecLayout::kReorth] = 0.0;
    rec[RecLayout::kFirst] = -1.0;
    st->reorth = 0;
  }
  const int hoff = RecLayout{s, 0}.h();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double rhs[kMaxS], h[kMaxS];
    for (int l = 0; l < s; ++l) rhs[l] = scratch[i * s + l];
    gram_solve_dev(grams[i], rhs, h);
    for (int l = 0; l < s; ++l) {
      rec[hoff + i * s + l] = h[l];
      coef[cH + i * s + l] = -h[l];
    }
  }
}

// nu = ||seed|| and the invariant-subspace test (sstep.hpp:315-324)
__global__ void k_arn_s2(ArnState* st, int k, double* rec, double* coef, const double* partials, int G, int dSeed,
                         int cInv) {
  SKC_PDL_ENTRY();
  if (arn_skip(st)) return;
  __shared__ double v[1];
  reduce_dots_dev(partials, G, dSeed, 1, v);
  if (threadIdx.x == 0) {
    const double nu = sqrt(v[0]);
    const double zn = rec[RecLayout::kZn];
    rec[RecLayout::kNu] = nu;
    if (nu <= 1e-14 * zn) {
      rec[RecLayout::kInv] = 1.0;
      st->status = kArnInvariant;
      st->block = k;
      st->halt = 1;
      return;
    }
    coef[cInv] = 1.0 / nu;
  }
}

// needs_reorth (sstep.hpp:401-414) on the device-computed cross products
__global__ void k_arn_check(ArnState* st, const Gram* grams, int k, double* rec, const double* partials, int G,
                            int dCross, int dWa, int s, double orth_tol, double* scratch) {
  SKC_PDL_ENTRY();
  if (arn_skip(st)) return;
  // (k <= 64 blocks: m is limited to 64)
  reduce_dots_dev(partials, G, dCross, k * s * s, scratch);
  __shared__ double sW[kMaxS * kMaxS];
  __shared__ int exceed[128];
  reduce_dots_dev(partials, G, dWa, s * s, sW);
  double cn2 = 0.0;  // sum_jc ||cand_jc||^2 in the reference's order (sstep.hpp:403)
  for (int jc = 0; jc < s; ++jc) cn2 += sW[jc * s + jc];
  // every block's test evaluated in parallel (same per-block arithmetic order), first hit wins
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double* cr = scratch + i * s * s;
    double acc = 0.0;
    for (int q = 0; q < s * s; ++q) acc += cr[q] * cr[q];
    exceed[i] = sqrt(acc) > orth_tol * sqrt(sd_trace(grams[i].w, s)) * sqrt(cn2);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int first = -1;
    for (int i = 0; i < k; ++i)
      if (exceed[i]) {
        first = i;
        break;
      }
    rec[RecLayout::kFirst] = first;
    rec[RecLayout::kReorth] = first >= 0 ? 1.0 : 0.0;
    st->reorth = first >= 0;
  }
}

// ---------------------------------------------------------------- on-chip block orthogonalization
// One kernel for a whole block iteration (sstep.hpp:297-379) when the candidate columns
// cand[:,1:] of every CTA's point slice fit in its shared memory: one CTA per SM owns points
// [b*P, (b+1)*P) and keeps its slice of the candidate there for
//   z = A v, the Scalar1 products and solves, the seed and nu, the candidate powers,
//   pass 0: k rounds  (Scalar2 solve in every CTA, cand -= V_i t, products V_{i+1}^T cand),
//   the cross products [V_0..V_{k-1}, cand]^T cand and the reorthogonalization test,
//   pass 1 (only when the test fires): V_0^T cand, k more rounds (t accumulated), W = cand^T cand,
// separated by grid-wide barriers; cand[:,1:] is written back once at the end.  Only the basis
// blocks stream from memory, and they stream through the TMA engine: a producer thread walks
// the launch's fixed schedule of (basis block, tile) jobs and issues one cp.async.bulk per column
// of a tile into a ring of shared-memory stages (full / empty mbarriers per stage); the 16
// consumer warps wait on a stage, compute from shared memory and release it with one arrive
// per warp.  The producer attends neither the CTA barriers nor the grid barriers, so the next
// phase's first tiles are in place during every reduce-and-solve and every grid barrier.
// (Measured on C2: a bulk copy costs the TMA unit ~85 ns whatever its size up to a few KB, so
// tiles are as large as the ring allows; the loaded latency of a copy is ~0.4 us, ~48 KB in
// flight per SM saturate the rate, and an L2 prefetch ahead of the copies lost.)
// Every CTA reduces the per-CTA partials in the same fixed order, so all CTAs take identical
// coefficients and the same reorthogonalization decision; CTA 0 writes the records and the
// device flags.
constexpr int ORTH_NT = 512;                 // consumer threads (16 warps)
constexpr int ORTH_THREADS = ORTH_NT + 32;   // + the producer warp
#ifndef SKC_ORTH_U
#define SKC_ORTH_U 2
#endif
constexpr int ORTH_U = SKC_ORTH_U;           // points per consumer thread per tile
constexpr int ORTH_T = ORTH_U * ORTH_NT;     // points per tile (point p stays with thread p mod 512)
constexpr int kOrthMaxStages = 8;
// cross products beyond this many are reduced once in the grid and published (one more grid
// barrier) instead of in every CTA.  Measured on C2 (one box, SKC_ORTH_OWNER_DOTS = off / 96 /
// 64 / 32 / 0): 4097 / 4144 / 4147 / 4157 / 4163 s-steps/s; the reorthogonalization test at
// k = 9 (160 products) 14.8 -> 4.0 us.
#ifndef SKC_ORTH_OWNER_DOTS
#define SKC_ORTH_OWNER_DOTS 32
#endif
constexpr int kOrthOwnerDots = SKC_ORTH_OWNER_DOTS;
constexpr size_t kOrthSmemCap = 226 * 1024;  // <= the 227 KB per-block limit less the static part
// candidate columns kept in shared memory (the rest in their basis slots, read back through a
// register prefetch): what is left of the 227 KB holds the ring's stages
#ifndef SKC_ORTH_SMEM_COLS
#define SKC_ORTH_SMEM_COLS 2
#endif
constexpr int kOrthSmemCols = SKC_ORTH_SMEM_COLS;
// reduced-product capacity: the cross test needs (k+1) s^2, a round s(s-1), Scalar1 k s + 1
__host__ __device__ inline int orth_prod_cap(int k, int s) { return ((k + 1) * s * s + 2) & ~1; }
__host__ __device__ inline int orth_h_cap(int k, int s) { return (k * s + 1) & ~1; }

// What a block's Scalar solves and the reorthogonalization test need of its GramSolver, in
// shared memory: the Cholesky factor and trace(W) (an LDL^T-factored block -- a failed
// Cholesky attempt, rare -- is solved from the full record in global memory)
template <int S>
struct GramC {
  double trace;
  int used_ldlt, pad;
  double fac[S * S];
};

struct OrthDesc {
  int s, k, build_next;
  int nst;                // stages of the basis ring
  int hint;               // L2 policy of the basis copies: 0 none, 1 evict_last, 2 evict_normal, 3 evict_first
  int64_t n, P;           // points, points per CTA
  DevOp op;
  const double* vin;      // v_{k-1}^{s-1}: z = A vin
  double* z;
  double* seed;
  const double* V;        // basis: block i column l at V + (i*s + l)*np
  int64_t np;
  const double* cand0;    // candidate column 0 (= cand[0] below, written by the powers phase)
  double* cand[kMaxS];    // candidate columns 0..s-1 of block slot k
  double* partials;
  int dz, dseed, dr0, dr1, dcross, dwb;
  Gram* grams;
  double* rec;            // this block iteration's record
  double* rec_push;       // the previous block iteration's record (its push_block)
  int rec_t, rec_h, rec_wraw;
  ArnState* st;
  double orth_tol;
  unsigned long long* trace;  // optional phase timestamps (CTA 0), diagnostics
  // level-by-level candidate powers on the slice extended by ghost rows (2D constant stencil,
  // the ghost rows fit the ring's stages); spow 0 = per-level sweeps with grid barriers
  int spow;
  double* reduced;  // published reductions of the wide cross products ((k+1) s^2 doubles)
  int owner_dots;   // cross products beyond this many are reduced once in the grid and published
};

// per-CTA completion time of a phase (diagnostics): slot base + CTA index
__device__ __forceinline__ void orth_mark_all(const OrthDesc& d, int base) {
  if (d.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    d.trace[base + blockIdx.x] = t;
  }
}

__device__ __forceinline__ void orth_mark(const OrthDesc& d, int slot) {
  if (d.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    d.trace[slot] = t;
  }
}

// barrier of the 512 consumer threads (named barrier 1: the producer warp does not attend)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(ORTH_NT) : "memory"); }

// Grid-wide barrier of the consumer threads: one monotonic counter (never reset: every CTA
// passes every barrier, so arrivals [g G, (g+1) G) belong to barrier g), one atomic per CTA,
// acquire polling.  The launch is cooperative, so all CTAs are resident.
// (Measured on C2: publishing each generation in a separate release word that the waiters poll
// -- arrivals then do not queue behind the pollers of the counter's line -- costs a third
// round trip per barrier and is 3% slower end to end: 4032 against 4165 s-steps/s.)
__device__ __forceinline__ void orth_gsync(unsigned long long* bar, unsigned G) {
  csync();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(bar, 1ull);
    const unsigned long long target = (old / G + 1) * G;
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    } while (v < target);
    __threadfence();
  }
  csync();
}

// reduce_dots_dev for the consumer threads (ungrouped partials; ends with csync)
__device__ __forceinline__ void orth_reduce(const double* __restrict__ partials, int G, int d0, int nd, double* out) {
  int tpd = 32;
  while (tpd > 1 && (ORTH_NT / tpd) < nd) tpd >>= 1;
  const int groups = ORTH_NT / tpd;
  const int grp = threadIdx.x / tpd, sub = threadIdx.x % tpd;
  for (int d = grp; d - grp < nd; d += groups) {  // uniform trip count across the warp
    double s = 0.0;
    if (d < nd) {
      const double* p = partials + (int64_t)(d0 + d) * kPartialPitch;
      // eight loads in flight per lane (the wide cross-product reductions are latency chains)
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int g = sub;
      for (; g + 7 * tpd < G; g += 8 * tpd) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + g + u * tpd);
        a0 += v[0];
        a1 += v[1];
        a2 += v[2];
        a3 += v[3];
        a0 += v[4];
        a1 += v[5];
        a2 += v[6];
        a3 += v[7];
      }
      for (; g + 3 * tpd < G; g += 4 * tpd) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(p + g + u * tpd);
        a0 += v[0];
        a1 += v[1];
        a2 += v[2];
        a3 += v[3];
      }
      for (; g < G; g += tpd) a0 += __ldcg(p + g);
      s = (a0 + a1) + (a2 + a3);
    }
    for (int o = tpd >> 1; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, tpd);
    if (sub == 0 && d < nd) out[d] = s;
  }
  csync();
}

// fixed-order CTA reduction of K per-thread accumulators into partial column blockIdx.x
template <int K>
__device__ __forceinline__ void orth_store(const double (&acc)[K], double* red, double* partials, int d0) {
  constexpr int NW = ORTH_NT / 32;
  const int warp = threadIdx.x >> 5;
  warp_sums(acc, red + warp * K);
  csync();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w * K + threadIdx.x];
    partials[(int64_t)(d0 + threadIdx.x) * kPartialPitch + blockIdx.x] = s;
  }
  csync();
}

// ring position: stage index and the parity of its current use
struct OrthRing {
  int idx;
  uint32_t ph;
  __device__ __forceinline__ void next(int nst) {
    if (++idx == nst) idx = 0, ph ^= 1u;
  }
};

template <int S>
__global__ void __launch_bounds__(ORTH_THREADS, 1) k_arn_step(const __grid_constant__ OrthDesc d) {
  SKC_PDL_ENTRY();
  constexpr int NC = S - 1;
  constexpr int T = ORTH_T, U = ORTH_U, NT = ORTH_NT;
  constexpr int SC = NC < kOrthSmemCols ? NC : kOrthSmemCols;  // candidate columns 1..SC on chip
  constexpr int NG = NC - SC;                                   // columns SC+1..s-1 in memory
  constexpr int NG1 = NG > 0 ? NG : 1;
  extern __shared__ __align__(16) double dsm[];
  // coefficients -t [s(s-1), 64] | -h [k s] | reduced products [(k+1) s^2] | the pushed block's
  // full GramSolver | compact Gram records of the k blocks | reduction scratch [16 warps][s^2]
  // | candidate slice [SC][P] | ring stages [nst][s][T]
  // (carved with pointer arithmetic on the shared array only -- an integer round trip would make
  // every derived pointer generic and turn the hot loops' LDS into generic loads; the candidate
  // slice and the stages are bulk-copy destinations: 16-byte aligned = an even double offset)
  double* tc = dsm;
  double* hc = dsm + 64;
  double* prod = hc + orth_h_cap(d.k, S);
  int off = 64 + orth_h_cap(d.k, S) + orth_prod_cap(d.k, S);
  Gram* gs = reinterpret_cast<Gram*>(dsm + off);
  off += (int)(sizeof(Gram) / sizeof(double));
  GramC<S>* gk = reinterpret_cast<GramC<S>*>(dsm + off);
  off += d.k * (int)(sizeof(GramC<S>) / sizeof(double));
  double* red = dsm + off;
  off += (NT / 32) * (S * S);
  off = (off + 1) & ~1;
  double* sc = dsm + off;
  double* stg = sc + (int64_t)(SC > 0 ? SC : 1) * d.P;
  __shared__ __align__(8) uint64_t s_full[kOrthMaxStages], s_empty[kOrthMaxStages], s_ctl, s_go;
  __shared__ volatile int s_quit, s_dec;
  __shared__ int s_jp;
  __shared__ int exceed[64];
  __shared__ int s_first, s_push_ok;
  const int tid = threadIdx.x;
  const int NST = d.nst;
  const int64_t base = (int64_t)blockIdx.x * d.P;
  const int64_t rem = d.n - base;
  const int cnt = rem <= 0 ? 0 : (int)(rem < d.P ? rem : d.P);
  const int ntiles = (cnt + T - 1) / T;
  const unsigned G = gridDim.x;
  const int K = d.k;
  const int64_t np = d.np;
  auto colp = [&](int i, int l) { return d.V + ((int64_t)i * S + l) * d.np + base; };
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&s_empty[q], NT / 32);
    }
    mbar_init(&s_ctl, 1);
    mbar_init(&s_go, 1);
    s_quit = 0;
    s_dec = 0;
    s_jp = 0;
    mbar_fence_init();
  }
  __syncthreads();

  // ================================================================ producer (one thread)
  // The schedule is a fixed function of (k, build_next) up to the reorthogonalization decision:
  // Scalar1 products (blocks k-1..0) | seed (0..k-1) | round-0 products (block 0) | rounds
  // (V_i and V_{i+1} tile by tile) | cross products (k-1..0) | the second pass' round-0 products
  // and rounds.  The first tiles of the second pass are issued before its decision is known
  // (block 0 was the cross pass' last block, so they come from L2); unused ones are drained by
  // the consumers before the CTA exits, as is whatever is in flight when the block iteration
  // stops early (s_quit).  Between the seed and the round-0 products the copies wait for the
  // powers phase (s_go): its ghost rows live in the ring's stages.
  if (tid >= NT) {
    if (tid != NT) return;
    OrthRing pp{0, 0u};
    int jp = 0;
    const uint64_t pol = d.hint == 1 ? policy_evict_last() : d.hint == 3 ? policy_evict_first() : policy_evict_normal();
    auto issue = [&](const double* blk, int t) -> bool {
      while (!mbar_try_wait(&s_empty[pp.idx], pp.ph ^ 1u))
        if (s_quit) return false;
      const int npts = cnt - t * T < T ? cnt - t * T : T;
      const uint32_t bytes = (uint32_t)((npts + 1) & ~1) * 8u;
      mbar_arrive_expect_tx(&s_full[pp.idx], S * bytes);
      double* dst = stg + (int64_t)pp.idx * (S * T);
      const double* src = blk + (int64_t)t * T;
#pragma unroll
      for (int l = 0; l < S; ++l) {
        if (d.hint)
          bulk_g2s_hint(dst + l * T, src + l * np, bytes, &s_full[pp.idx], pol);
        else
          bulk_g2s(dst + l * T, src + l * np, bytes, &s_full[pp.idx]);
      }
      pp.next(NST);
      ++jp;
      return true;
    };
    auto sweep = [&](int i, int t0) -> bool {
      const double* b = colp(i, 0);
      for (int t = t0; t < ntiles; ++t)
        if (!issue(b, t)) return false;
      return true;
    };
    auto produce = [&]() {
      for (int i = K - 1; i >= 0; --i)
        if (!sweep(i, 0)) return;
      for (int i = 0; i < K; ++i)
        if (!sweep(i, 0)) return;
      if (!d.build_next) return;
      while (!mbar_try_wait(&s_go, 0u))  // the powers phase owns the ring until then
        if (s_quit) return;
      for (int pass = 0; pass < 2; ++pass) {
        // (the second pass has no round-0 product sweep: its V_0^T cand are the cross products)
        if (pass == 0 && !sweep(0, 0)) return;
        int spec = pass == 1 ? NST : -1;  // second pass: copies issued before its decision is known
        for (int i = 0; i < K; ++i) {
          const double* bi = colp(i, 0);
          const double* bn = colp(i + 1 < K ? i + 1 : i, 0);
          for (int t = 0; t < ntiles; ++t) {
            for (int h = 0; h < (i + 1 < K ? 2 : 1); ++h) {
              if (spec == 0) {
                int dec;
                while ((dec = s_dec) == 0)
                  if (s_quit) return;
                if (dec == 1) return;
              }
              if (spec >= 0) --spec;
              if (!issue(h ? bn : bi, t)) return;
            }
          }
        }
        if (spec >= 0) {  // (fewer jobs than stages: still stop on a negative decision)
          int dec;
          while ((dec = s_dec) == 0)
            if (s_quit) return;
          if (dec == 1) return;
        }
        if (pass == 0)
          for (int i = K - 1; i >= 0; --i)
            if (!sweep(i, 0)) return;
      }
    };
    produce();
    s_jp = jp;
    mbar_arrive(&s_ctl);
    return;
  }

  // ================================================================ consumers
  OrthRing pc{0, 0u};
  int jc = 0;
  const int lane = tid & 31;
  // wait for the next job's stage / release it
  auto cwait = [&]() -> const double* {
    mbar_wait(&s_full[pc.idx], pc.ph);
    return stg + (int64_t)pc.idx * (S * T) + tid;
  };
  auto crel = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[pc.idx]);
    pc.next(NST);
    ++jc;
  };
  // leave the kernel: stop the producer and wait for the copies still in flight
  auto finish = [&]() {
    csync();
    if (tid == 0) {
      s_quit = 1;
      mbar_wait(&s_ctl, 0u);
      const int jp = s_jp;
      for (; jc < jp; ++jc) {
        mbar_wait(&s_full[pc.idx], pc.ph);
        pc.next(NST);
      }
    }
  };
  // this slice of candidate column j+1 (j = 0..s-2): the first SC in shared memory, the rest in
  // their basis slots in global memory
  // (slots in reverse order: column 1 in the last slot, so that slot 0 -- z, the seed and level 0
  // of the powers -- is not written before level 1 is complete)
  auto ccol = [&](int j) -> double* { return j < SC ? sc + (int64_t)(SC - 1 - j) * d.P : d.cand[j + 1] + base; };
  // in-memory candidate column g (candidate column SC+1+g), this slice
  auto gcol = [&](int g) -> double* { return d.cand[SC + 1 + g] + base; };

  // W_i x = rhs for basis block i (Cholesky factor from shared memory; LDL^T-factored blocks
  // from the full record)
  auto bsolve = [&](int i, const double* rhs, double* x) {
    if (S == 1 || gk[i].used_ldlt) {
      double r2[kMaxS], x2[kMaxS];
#pragma unroll
      for (int q = 0; q < S; ++q) r2[q] = rhs[q];
      gram_solve(i == K - 1 && K >= 2 ? *gs : d.grams[i], r2, x2);
#pragma unroll
      for (int q = 0; q < S; ++q) x[q] = x2[q];
    } else {
      chol_solve_t<S>(gk[i].fac, rhs, x);
    }
  };

  // Scalar2 for block i from partials src: every CTA solves W_i t = V_i^T cand[:,1:]
  // (src < 0: the products are block 0 of the reduced cross products already in prod, [l][jc])
  auto scalar = [&](int i, int src, int accumulate) {
    if (src >= 0) orth_reduce(d.partials, (int)G, src, S * NC, prod);  // ends with csync
    if (tid < NC) {
      const int jcl = tid;
      double rhs[kMaxS], t[kMaxS];
#pragma unroll
      for (int l = 0; l < S; ++l) rhs[l] = src >= 0 ? prod[l * NC + jcl] : prod[l * S + jcl + 1];
      bsolve(i, rhs, t);
#pragma unroll
      for (int l = 0; l < S; ++l) {
        tc[l * NC + jcl] = -t[l];
        if (blockIdx.x == 0) {
          double* ta = d.rec + d.rec_t + i * S * S + l * S + (jcl + 1);
          *ta = accumulate ? *ta + t[l] : t[l];
        }
      }
    }
    csync();
  };

  // the in-memory candidate columns of tile t's points of this thread (issued a tile ahead)
  auto gload = [&](int t, double (&o)[U][NG1]) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const int p = t * T + u * NT + tid;
        o[u][g] = p < cnt ? __ldcg(gcol(g) + p) : 0.0;
      }
  };

  // cand[:,1:] -= V_i t ; products V_{i+1}^T cand[:,1:] -> partials dst (when i+1 < k).  Point
  // p stays with thread p mod 512 and tiles go in ascending order, so the products accumulate
  // in ascending point order per thread.
  auto round = [&](int i, int dst, bool wb, auto&& pre) {
    const bool dots = i + 1 < d.k;
    double acc[S * NC];
#pragma unroll
    for (int q = 0; q < S * NC; ++q) acc[q] = 0.0;
    double gc[U][NG1], gn[U][NG1];
    gload(0, gc);
    pre();
    for (int t = 0; t < ntiles; ++t) {
      gload(t + 1, gn);
      double cv[U][NC];
      {
        const double* sp = cwait();
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = t * T + u * NT + tid;
          const bool has = p < cnt;
#pragma unroll
          for (int j = 0; j < SC; ++j) cv[u][j] = has ? ccol(j)[p] : 0.0;
#pragma unroll
          for (int g = 0; g < NG; ++g) cv[u][SC + g] = gc[u][g];
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double v = sp[l * T + u * NT];
#pragma unroll
            for (int j = 0; j < NC; ++j) cv[u][j] = dadd(cv[u][j], dmul(tc[l * NC + j], v));
          }
          if (has) {
#pragma unroll
            for (int j = 0; j < SC; ++j) ccol(j)[p] = cv[u][j];
#pragma unroll
            for (int g = 0; g < NG; ++g) gcol(g)[p] = cv[u][SC + g];
            if (wb) {  // (the columns past SC already live in their basis slots)
#pragma unroll
              for (int j = 0; j < SC; ++j) d.cand[j + 1][base + p] = cv[u][j];
            }
          }
        }
        crel();
      }
      if (dots) {
        const double* sp = cwait();
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (t * T + u * NT + tid < cnt) {
#pragma unroll
            for (int l = 0; l < S; ++l) {
              const double w = sp[l * T + u * NT];
#pragma unroll
              for (int j = 0; j < NC; ++j) acc[l * NC + j] = fma(w, cv[u][j], acc[l * NC + j]);
            }
          }
        }
        crel();
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < NG; ++g) gc[u][g] = gn[u][g];
    }
    if (dots) orth_store(acc, red, d.partials, dst);
  };

  // round-0 products V_0^T cand[:,1:] -> partials dr0 (sstep.hpp:341)
  auto r0_products = [&]() {
    double acc[S * NC];
#pragma unroll
    for (int q = 0; q < S * NC; ++q) acc[q] = 0.0;
    double gc[U][NG1], gn[U][NG1];
    gload(0, gc);
    for (int t = 0; t < ntiles; ++t) {
      gload(t + 1, gn);
      const double* sp = cwait();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = t * T + u * NT + tid;
        if (p < cnt) {
          double cv[NC];
#pragma unroll
          for (int j = 0; j < SC; ++j) cv[j] = ccol(j)[p];
#pragma unroll
          for (int g = 0; g < NG; ++g) cv[SC + g] = gc[u][g];
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double lv = sp[l * T + u * NT];
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[l * NC + j] = fma(lv, cv[j], acc[l * NC + j]);
          }
        }
      }
      crel();
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < NG; ++g) gc[u][g] = gn[u][g];
    }
    orth_store(acc, red, d.partials, d.dr0);
  };

  // L-block products with the full candidate: lhs(l) . cand[:,jc] for one block of s columns
  // (block i of the basis, or the candidate itself when i == k) -> partials d0 + l*s + jc.
  // Candidate column 0 and the columns past SC come from memory, issued a tile ahead.
  auto cross_block = [&](int i, int d0) {
    double acc[S * S];
#pragma unroll
    for (int q = 0; q < S * S; ++q) acc[q] = 0.0;
    const double* c0p = d.cand0 + base;
    const bool basis = i < d.k;
    double gc[U][1 + NG], gn[U][1 + NG];
    auto pfload = [&](int t, double (&o)[U][1 + NG]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = t * T + u * NT + tid;
        o[u][0] = p < cnt ? __ldcg(c0p + p) : 0.0;
#pragma unroll
        for (int g = 0; g < NG; ++g) o[u][1 + g] = p < cnt ? __ldcg(gcol(g) + p) : 0.0;
      }
    };
    pfload(0, gc);
    for (int t = 0; t < ntiles; ++t) {
      pfload(t + 1, gn);
      const double* sp = basis ? cwait() : nullptr;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = t * T + u * NT + tid;
        if (p < cnt) {
          double b[S];
          b[0] = gc[u][0];
#pragma unroll
          for (int j = 0; j < SC; ++j) b[1 + j] = ccol(j)[p];
#pragma unroll
          for (int g = 0; g < NG; ++g) b[1 + SC + g] = gc[u][1 + g];
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double av = basis ? sp[l * T + u * NT] : b[l];
#pragma unroll
            for (int jcl = 0; jcl < S; ++jcl) acc[l * S + jcl] = fma(av, b[jcl], acc[l * S + jcl]);
          }
        }
      }
      if (basis) crel();
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < 1 + NG; ++g) gc[u][g] = gn[u][g];
    }
    orth_store(acc, red, d.partials, d0);
  };

  // push_block of the previous block iteration's candidate (sstep.hpp:375, 392-399) runs here,
  // off the previous kernel's tail: every CTA reduces its W (from the pass that produced the
  // candidate) and factors it in the Scalar1 phase; CTA 0 records it and stores the factor
  const bool push = K >= 2;
  if (push)
    orth_reduce(d.partials, (int)G, __ldg(&d.st->reorth) ? d.dwb : d.dcross + (K - 1) * S * S, S * S, tc);
  // what the solves need of blocks 0..k-1 (k-2 with the push) into shared memory
  for (int w = tid; w < (push ? K - 1 : K) * (S * S + 1); w += NT) {
    const int i = w / (S * S + 1), q = w - i * (S * S + 1);
    const Gram& g = d.grams[i];
    if (q < S * S) {
      gk[i].fac[q] = g.fac[q];
    } else {
      gk[i].trace = sd_trace(g.w, S);
      gk[i].used_ldlt = g.used_ldlt;
    }
  }
  orth_mark(d, 39);
  auto apply_slice = [&](const double* x, const double* xs, double xscale, auto&& put) {
    if (d.op.kind == kStencilConst && d.op.dim == 2) {
      const int nx = (int)d.op.nx, ny = (int)d.op.ny;
      const double cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
      const double* xb = x + base;  // slice-relative view of x in memory
      auto get = [&](int o) {
        const double v = xs && o >= 0 && o < cnt ? xs[o] : xb[o];
        return xscale != 0.0 ? __dmul_rn(v, xscale) : v;
      };
      const uint32_t xs32 = xs ? smem_u32(xs) : 0u;
      auto gets = [&](int o) {  // (o inside the slice)
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(xs32 + 8u * (uint32_t)o));
        return xscale != 0.0 ? __dmul_rn(v, xscale) : v;
      };
      // four points per thread per iteration, every neighbour load issued before the sums
      constexpr int U = 4;
      int i[U], jr[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = base + tid + u * ORTH_NT;
        i[u] = (int)(q % nx), jr[u] = (int)(q / nx);
      }
      for (int p0 = tid; p0 < cnt; p0 += U * ORTH_NT) {
        double vs[U], vw[U], vc[U], ve[U], vn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = p0 + u * ORTH_NT;
          const bool in = p < cnt;
          if (xs && in && p >= nx && p + nx < cnt && i[u] > 0 && i[u] + 1 < nx) {
            // interior of the slice: every neighbour present and in shared memory
            vs[u] = gets(p - nx);
            vw[u] = gets(p - 1);
            vc[u] = gets(p);
            ve[u] = gets(p + 1);
            vn[u] = gets(p + nx);
          } else {
            vs[u] = in && jr[u] > 0 ? get(p - nx) : 0.0;
            vw[u] = in && i[u] > 0 ? get(p - 1) : 0.0;
            vc[u] = in ? get(p) : 0.0;
            ve[u] = in && i[u] + 1 < nx ? get(p + 1) : 0.0;
            vn[u] = in && jr[u] + 1 < ny ? get(p + nx) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = p0 + u * ORTH_NT;
          if (p < cnt) {
            double a = 0.0;
            if (jr[u] > 0) a = __dadd_rn(a, __dmul_rn(cS, vs[u]));
            if (i[u] > 0) a = __dadd_rn(a, __dmul_rn(cW, vw[u]));
            a = __dadd_rn(a, __dmul_rn(cC, vc[u]));
            if (i[u] + 1 < nx) a = __dadd_rn(a, __dmul_rn(cE, ve[u]));
            if (jr[u] + 1 < ny) a = __dadd_rn(a, __dmul_rn(cN, vn[u]));
            put(p, a, vc[u]);
          }
          i[u] += U * ORTH_NT;
          while (i[u] >= nx) i[u] -= nx, ++jr[u];
        }
      }
      return;
    }
    GridWalk w;
    if (tid < cnt) w.init(d.op, base + tid);
    auto fetch = [&](int64_t q) {
      const int64_t o = q - base;
      const double v = xs && o >= 0 && o < cnt ? xs[o] : x[q];
      return xscale != 0.0 ? __dmul_rn(v, xscale) : v;
    };
    for (int p = tid; p < cnt; p += ORTH_NT, w.step(d.op, ORTH_NT))
      put(p, apply_point(d.op, fetch, base + p, w), fetch(base + p));
  };
  // z and seed of this slice stay in shared memory (slot 0, free until the powers reach it)
  double* zs = sc;
  apply_slice(d.vin, nullptr, 0.0, [&](int p, double v, double) { zs[p] = v; });
  orth_mark(d, 40);
  // ---- Scalar1 products V_i^T z (i < k) -> dz + i s + l, and z.z -> dz + k s (each thread
  //      reads back its own z); blocks in descending order, so the seed sweep's first blocks
  //      are still in L2
  {
    double zz[1] = {0.0};
    for (int i = K - 1; i >= 0; --i) {
      double acc[S];
#pragma unroll
      for (int q = 0; q < S; ++q) acc[q] = 0.0;
      for (int t = 0; t < ntiles; ++t) {
        const double* sp = cwait();
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = t * T + u * NT + tid;
          if (p < cnt) {
            const double zv = zs[p];
#pragma unroll
            for (int l = 0; l < S; ++l) acc[l] = fma(sp[l * T + u * NT], zv, acc[l]);
            if (i == 0) zz[0] = fma(zv, zv, zz[0]);
          }
        }
        crel();
      }
      orth_store(acc, red, d.partials, d.dz + i * S);
    }
    orth_store(zz, red, d.partials, d.dz + K * S);
  }
  orth_mark(d, 6);
  orth_mark_all(d, 256);
  // the halt flag (raised by an earlier block step, or by the side stream's least-squares
  // kernel, possibly while this grid was being scheduled) as CTA 0 sees it now, made the whole
  // grid's decision by the barrier
  if (blockIdx.x == 0 && tid == 0) d.st->hseen = *reinterpret_cast<const volatile int*>(&d.st->halt);
  orth_gsync(&d.st->gbar, G);
  if (*reinterpret_cast<const volatile int*>(&d.st->hseen)) {
    finish();
    return;
  }
  // ---- Scalar1 (sstep.hpp:301-310): zn, h_i = W_i^{-1} V_i^T z in every CTA (Gram factors
  // from shared memory); CTA 0 records
  orth_reduce(d.partials, (int)G, d.dz, K * S + 1, prod);  // (ends with csync)
  if (push) {
    if (tid == 0) {
      const bool ok = arn_push_body<S>(d.st, *gs, K - 1, d.rec_push, tc, S, blockIdx.x == 0);
      s_push_ok = ok;
      if (ok) {
#pragma unroll
        for (int q = 0; q < S * S; ++q) gk[K - 1].fac[q] = gs->fac[q];
        gk[K - 1].trace = sd_trace(gs->w, S);
        gk[K - 1].used_ldlt = gs->used_ldlt;
        if (blockIdx.x == 0) d.grams[K - 1] = *gs;
      }
    }
    csync();
    if (!s_push_ok) {  // basis collapse (identical decision in every CTA)
      finish();
      return;
    }
  }
  const double zn = sqrt(prod[K * S]);
  if (blockIdx.x == 0 && tid == 0) {
    d.rec[RecLayout::kZn] = zn;
    d.rec[RecLayout::kReorth] = 0.0;
    d.rec[RecLayout::kFirst] = -1.0;
  }
  for (int i = tid; i < K; i += ORTH_NT) {
    double rhs[kMaxS], h[kMaxS];
#pragma unroll
    for (int l = 0; l < S; ++l) rhs[l] = prod[i * S + l];
    bsolve(i, rhs, h);
#pragma unroll
    for (int l = 0; l < S; ++l) {
      hc[i * S + l] = -h[l];
      if (blockIdx.x == 0) d.rec[d.rec_h + i * S + l] = h[l];
    }
  }
  csync();
  orth_mark(d, 41);
  // ---- seed = z - sum_i V_i h_i (terms in block order, multiply and add rounded separately),
  //      one sweep per block with the running sum in shared memory (every point stays with
  //      its thread), then ||seed||^2
  {
    for (int i = 0; i < K; ++i) {
      double hl[S];
#pragma unroll
      for (int l = 0; l < S; ++l) hl[l] = hc[i * S + l];
      for (int t = 0; t < ntiles; ++t) {
        const double* sp = cwait();
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int p = t * T + u * NT + tid;
          if (p < cnt) {
            double o = zs[p];
#pragma unroll
            for (int l = 0; l < S; ++l) o = dadd(o, dmul(hl[l], sp[l * T + u * NT]));
            zs[p] = o;
          }
        }
        crel();
      }
    }
    double acc[1] = {0.0};
    for (int p = tid; p < cnt; p += ORTH_NT) {
      const double o = zs[p];
      d.seed[base + p] = o;
      acc[0] = fma(o, o, acc[0]);
    }
    orth_store(acc, red, d.partials, d.dseed);
  }
  orth_mark(d, 7);
  orth_mark_all(d, 512);
  orth_gsync(&d.st->gbar, G);
  // ---- nu = ||seed|| and the invariant-subspace test (sstep.hpp:315-324)
  orth_reduce(d.partials, (int)G, d.dseed, 1, prod);
  const double nu = sqrt(prod[0]);
  if (blockIdx.x == 0 && tid == 0) d.rec[RecLayout::kNu] = nu;
  if (nu <= 1e-14 * zn) {  // identical decision in every CTA
    if (blockIdx.x == 0 && tid == 0) {
      d.rec[RecLayout::kInv] = 1.0;
      d.st->status = kArnInvariant;
      d.st->block = K;
      d.st->halt = 1;
    }
    finish();
    return;
  }
  const double inv = 1.0 / nu;
  orth_mark(d, 42);
  // ---- candidate block [v, A v, .., A^{s-1} v], v = seed / nu (krylov_block, block.hpp:59-67):
  //      every level is an exact spmv of the previous one; levels 1..s-1 stay on chip (or in
  //      their basis slots), levels 0..s-2 also go to memory for the neighbours' next level
  orth_mark(d, 44);
  if (d.spow == 2) {
    // Row-aligned slices (P a multiple of nx; host: 2D constant stencil, nx even, nx <= 2 x 512
    // threads, the ghost rows fit the ring): level by level over the slice's grid rows extended
    // by e_j = s-1-j rows on each side (level j is needed that far for the slice's last level),
    // redundantly with the neighbouring CTAs, so no level needs another CTA's results and CTA
    // barriers suffice.  Every level lives in shared memory: the slice rows in the candidate's
    // column slots (level 0 = seed / nu in slot 0, which is next written after level 1 is
    // done), the ghost rows in the idle ring (two regions used alternately).  A thread owns a
    // column pair: it reads its pair of the rows r-1, r, r+1 of the previous level as 16-byte
    // loads and takes the W / E neighbours from the adjacent lanes (shared memory at the warp
    // edges).  Each point is the same ascending-column sum as spmv (absent neighbours skipped),
    // so the levels are bit-identical to successive sweeps.
    const int nx = (int)d.op.nx, ny = (int)d.op.ny;
    const double cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
    const int R0 = (int)(base / nx), Rs = cnt / nx;
    double* regA = stg;
    double* regB = stg + 2 * (S - 1) * nx;
    // row r (grid row) of level j, inside the level's extended range
    auto rowp = [&](int j, int r) -> double* {
      const int rr = r - R0, e = S - 1 - j;
      if (rr >= 0 && rr < Rs) return (j == 0 ? zs : ccol(j - 1)) + rr * nx;
      double* g = (j & 1) ? regB : regA;
      return rr < 0 ? g + (rr + e) * nx : g + (e + rr - Rs) * nx;
    };
    const int c0 = 2 * tid;
    const bool act = c0 < nx;
    if (cnt > 0) {
      // level 0: the slice in place (and to memory), its ghost rows from the seed in memory
      for (int p = tid; p < cnt; p += NT) {
        const double v0 = __dmul_rn(zs[p], inv);
        zs[p] = v0;
        d.cand[0][base + p] = v0;
      }
      // (ghost index g: e0 rows below the slice, then e0 rows above it; GU loads in flight --
      // the six ghost rows of C2 in two round trips)
      constexpr int GU = 6;
      const int e0 = S - 1, half = e0 * nx;
      for (int g0 = tid; g0 < 2 * half; g0 += GU * NT) {
        double v[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int g = g0 + u * NT;
          const int w = g < half ? g : g - half;
          const int r = (g < half ? R0 - e0 : R0 + Rs) + w / nx;
          v[u] = g < 2 * half && r >= 0 && r < ny ? __ldcg(d.seed + (int64_t)r * nx + w % nx) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u)
          if (g0 + u * NT < 2 * half) regA[g0 + u * NT] = __dmul_rn(v[u], inv);
      }
    }
    csync();
    orth_mark(d, 45);
    if (cnt > 0) {
#pragma unroll
      for (int j = 1; j < S; ++j) {
        if (j > 1) orth_mark(d, 44 + 2 * j - 1);
        const int e = S - 1 - j;
        const int rlo = R0 - e < 0 ? 0 : R0 - e, rhi = R0 + Rs + e > ny ? ny : R0 + Rs + e;
        // (rows r-1, r, r+1 of the previous level slide through registers: one 16-byte load per
        // row, issued a row ahead of its first use)
        auto ldrow = [&](int r) -> double2 {
          return act && r >= 0 && r < ny ? *reinterpret_cast<const double2*>(rowp(j - 1, r) + c0)
                                         : make_double2(0.0, 0.0);
        };
        double2 Sv = ldrow(rlo - 1), C = ldrow(rlo), Nv = ldrow(rlo + 1);
        for (int r = rlo; r < rhi; ++r) {
          const bool hs = r > 0, hn = r + 1 < ny;
          const double* pc = rowp(j - 1, r);
          const double2 NN = r + 1 < rhi ? ldrow(r + 2) : make_double2(0.0, 0.0);
          double w0 = __shfl_up_sync(0xffffffffu, C.y, 1);
          double e1 = __shfl_down_sync(0xffffffffu, C.x, 1);
          if (act) {
            if (lane == 0 && c0 > 0) w0 = pc[c0 - 1];
            if (lane == 31 && c0 + 2 < nx) e1 = pc[c0 + 2];
            double a0 = 0.0, a1 = 0.0;
            if (hs) {
              a0 = __dadd_rn(a0, __dmul_rn(cS, Sv.x));
              a1 = __dadd_rn(a1, __dmul_rn(cS, Sv.y));
            }
            if (c0 > 0) a0 = __dadd_rn(a0, __dmul_rn(cW, w0));
            a1 = __dadd_rn(a1, __dmul_rn(cW, C.x));
            a0 = __dadd_rn(a0, __dmul_rn(cC, C.x));
            a1 = __dadd_rn(a1, __dmul_rn(cC, C.y));
            a0 = __dadd_rn(a0, __dmul_rn(cE, C.y));
            if (c0 + 2 < nx) a1 = __dadd_rn(a1, __dmul_rn(cE, e1));
            if (hn) {
              a0 = __dadd_rn(a0, __dmul_rn(cN, Nv.x));
              a1 = __dadd_rn(a1, __dmul_rn(cN, Nv.y));
            }
            *reinterpret_cast<double2*>(rowp(j, r) + c0) = make_double2(a0, a1);
            if (!d.build_next && j - 1 < SC && r >= R0 && r < R0 + Rs)
              *reinterpret_cast<double2*>(d.cand[j] + (int64_t)r * nx + c0) = make_double2(a0, a1);
          }
          Sv = C, C = Nv, Nv = NN;
        }
        csync();
        orth_mark(d, 44 + 2 * j);
      }
    } else {
#pragma unroll
      for (int j = 1; j < S; ++j) csync();
    }
  } else
  if (d.spow) {
    // Level by level over the slice extended by e_j = s-1-j index rows of nx points on each side
    // (level j is needed that far for the slice's last level), redundantly with the neighbouring
    // CTAs, so no level needs another CTA's results and CTA barriers suffice.  Every level lives
    // in shared memory: the slice part in the candidate's column slots (level 0 = seed / nu in
    // the slot of the last on-chip column, which is written after level 1 is done), the ghost
    // parts in the idle ring (two regions used alternately).  With a single on-chip column
    // (s = 2) level 1 reads seed / nu from memory instead.  Each point is the same
    // ascending-column sum as spmv, so the levels are bit-identical to successive sweeps.
    // (Host: 2D constant stencil, n < 2^30, the ghost rows fit the ring.)
    constexpr bool L0S = SC >= 2;
    const int nx = (int)d.op.nx, ny = (int)d.op.ny;
    const double cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
    const int b32 = (int)base, n32 = (int)d.n;
    double* regA = stg;
    double* regB = stg + 2 * (S - 1) * nx;
    // level j at slice-relative index v inside its extended range
    auto ext = [&](int j, int v) -> double* {
      if ((unsigned)v < (unsigned)cnt) return j == 0 ? zs + v : ccol(j - 1) + v;
      const int e = S - 1 - j;
      double* g = (j & 1) ? regB : regA;
      return v < 0 ? g + (v + e * nx) : g + (e * nx + (v - cnt));
    };
    if (L0S && cnt > 0) {
      // level 0: the slice in place (and to memory), its ghost rows from the seed in memory
      for (int p = tid; p < cnt; p += NT) {
        const double v0 = __dmul_rn(zs[p], inv);
        zs[p] = v0;
        d.cand[0][base + p] = v0;
      }
      const int e0 = S - 1;
      const int glo = b32 - e0 * nx < 0 ? -b32 : -e0 * nx;
      const int ghi = b32 + cnt + e0 * nx > n32 ? n32 - b32 : cnt + e0 * nx;
      for (int v = glo + tid; v < 0; v += NT) *ext(0, v) = __dmul_rn(__ldcg(d.seed + (b32 + v)), inv);
      for (int v = cnt + tid; v < ghi; v += NT) *ext(0, v) = __dmul_rn(__ldcg(d.seed + (b32 + v)), inv);
    }
    if (L0S) csync();
    orth_mark(d, 45);
    if (cnt > 0) {
#pragma unroll
      for (int j = 1; j < S; ++j) {
        if (j > 1) orth_mark(d, 44 + 2 * j - 1);
        const int e = S - 1 - j;
        int lo = -e * nx, hi = cnt + e * nx;
        if (b32 + lo < 0) lo = -b32;
        if (b32 + hi > n32) hi = n32 - b32;
        constexpr int UP = 2;  // points per thread in flight
        int ii[UP], jr[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int q = b32 + lo + tid + u * NT;
          ii[u] = q % nx, jr[u] = q / nx;
        }
        double* outs = ccol(j - 1);
        const double* ins = j == 1 ? zs : ccol(j > 1 ? j - 2 : 0);
        for (int v0 = lo + tid; v0 < hi; v0 += UP * NT) {
          double a[UP], x0[UP];
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const int v = v0 + u * NT;
            const bool in = v < hi;
            a[u] = 0.0;
            x0[u] = 0.0;
            if ((L0S || j > 1) && in && v >= nx && v + nx < cnt && ii[u] > 0 && ii[u] + 1 < nx) {
              // every neighbour present and inside the slice
              const double* pj = ins + v;
              double t = __dadd_rn(0.0, __dmul_rn(cS, pj[-nx]));
              t = __dadd_rn(t, __dmul_rn(cW, pj[-1]));
              x0[u] = pj[0];
              t = __dadd_rn(t, __dmul_rn(cC, x0[u]));
              t = __dadd_rn(t, __dmul_rn(cE, pj[1]));
              a[u] = __dadd_rn(t, __dmul_rn(cN, pj[nx]));
            } else if (in) {
              const bool hs = jr[u] > 0, hw = ii[u] > 0, he = ii[u] + 1 < nx, hn = jr[u] + 1 < ny;
              double xs_, xw_, xe_, xn_;
              if (!L0S && j == 1) {  // seed / nu from memory (the multiply rounded as when level 0 is stored)
                const double* sq = d.seed + (b32 + v);
                xs_ = hs ? __dmul_rn(sq[-nx], inv) : 0.0;
                xw_ = hw ? __dmul_rn(sq[-1], inv) : 0.0;
                x0[u] = __dmul_rn(sq[0], inv);
                xe_ = he ? __dmul_rn(sq[1], inv) : 0.0;
                xn_ = hn ? __dmul_rn(sq[nx], inv) : 0.0;
              } else {
                xs_ = hs ? *ext(j - 1, v - nx) : 0.0;
                xw_ = hw ? *ext(j - 1, v - 1) : 0.0;
                x0[u] = *ext(j - 1, v);
                xe_ = he ? *ext(j - 1, v + 1) : 0.0;
                xn_ = hn ? *ext(j - 1, v + nx) : 0.0;
              }
              double t = 0.0;
              if (hs) t = __dadd_rn(t, __dmul_rn(cS, xs_));
              if (hw) t = __dadd_rn(t, __dmul_rn(cW, xw_));
              t = __dadd_rn(t, __dmul_rn(cC, x0[u]));
              if (he) t = __dadd_rn(t, __dmul_rn(cE, xe_));
              if (hn) t = __dadd_rn(t, __dmul_rn(cN, xn_));
              a[u] = t;
            }
          }
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const int v = v0 + u * NT;
            if (v < hi) {
              if ((unsigned)v < (unsigned)cnt) {
                outs[v] = a[u];
                if (!L0S && j == 1) d.cand[0][base + v] = x0[u];
                if (!d.build_next && j - 1 < SC) d.cand[j][base + v] = a[u];
              } else {
                *ext(j, v) = a[u];
              }
            }
            ii[u] += UP * NT;
            while (ii[u] >= nx) ii[u] -= nx, ++jr[u];
          }
        }
        csync();
        orth_mark(d, 44 + 2 * j);
      }
    } else {
#pragma unroll
      for (int j = 1; j < S; ++j) csync();
    }
  } else
  // level 1 reads seed / nu on the fly (level 0 is stored by the same sweep); levels >= 2 read
  // their source from shared memory inside the slice
  for (int j = 1; j < S; ++j) {
    if (j > 1) orth_gsync(&d.st->gbar, G);
    orth_mark(d, 44 + 2 * j - 1);
    const bool to_mem = j + 1 < S || !d.build_next;
    apply_slice(j == 1 ? d.seed : d.cand[j - 1], j >= 2 && j - 2 < SC ? ccol(j - 2) : nullptr, j == 1 ? inv : 0.0,
                [&](int p, double v, double xc) {
                  if (j == 1) d.cand[0][base + p] = xc;
                  ccol(j - 1)[p] = v;
                  if (to_mem && j - 1 < SC) d.cand[j][base + p] = v;
                });
    orth_mark(d, 44 + 2 * j);
  }
  orth_mark(d, 43);
  if (!d.build_next) {  // the last block iteration builds the candidate only
    finish();
    return;
  }
  // the ring is the producer's again (the ghost rows are dead: every level ended with a barrier)
  fence_proxy_async();
  csync();
  if (tid == 0) mbar_arrive(&s_go);
  // ---- round-0 products V_0^T cand[:,1:] (sstep.hpp:341)
  r0_products();
  orth_gsync(&d.st->gbar, G);
  orth_mark(d, 0);
  // ---- pass 0; the last round also writes the candidate back (final unless a second pass runs)
  for (int i = 0; i < K; ++i) {
    round(i, ((i + 1) & 1) ? d.dr1 : d.dr0, i + 1 == K, [&] {
      scalar(i, (i & 1) ? d.dr1 : d.dr0, 0);
      orth_mark(d, 8 + 3 * i);
    });
    orth_mark(d, 9 + 3 * i);
    if (i + 1 < K) orth_gsync(&d.st->gbar, G);
    orth_mark(d, 10 + 3 * i);
  }
  orth_mark(d, 60);
  // ---- cross products and W (needs_reorth, sstep.hpp:401-414); blocks in descending order (the
  //      next seed sweep starts at block 0)
  for (int i = K; i >= 0; --i) cross_block(i, d.dcross + i * S * S);
  orth_mark(d, 1);
  orth_mark_all(d, 768);
  orth_gsync(&d.st->gbar, G);
  orth_mark(d, 2);
  if ((K + 1) * S * S > d.owner_dots) {
    // Wide cross products: reducing them in every CTA reads (k+1) s^2 x G partials G times over
    // (27.6 MB through L2 at k = 9 on C2, 13 us).  Instead warp w of the grid reduces product w
    // (lane partial sums over g = lane, lane + 32, .., then the shuffle tree: a fixed order),
    // publishes it, and after one more grid barrier every CTA loads the reduced values.
    const int nd = (K + 1) * S * S;
    const int warp = tid >> 5;
    for (int dd = (int)blockIdx.x * (NT / 32) + warp; dd < nd; dd += (int)G * (NT / 32)) {
      const double* p = d.partials + (int64_t)(d.dcross + dd) * kPartialPitch;
      double v[5];
#pragma unroll
      for (int u = 0; u < 5; ++u) v[u] = lane + 32 * u < (int)G ? __ldcg(p + lane + 32 * u) : 0.0;
      double a = ((v[0] + v[1]) + (v[2] + v[3])) + v[4];
      for (int g = lane + 160; g < (int)G; g += 32) a += __ldcg(p + g);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
      if (lane == 0) d.reduced[dd] = a;
    }
    orth_gsync(&d.st->gbar, G);
    for (int e = tid; e < nd; e += NT) prod[e] = __ldcg(d.reduced + e);
    csync();
  } else {
    orth_reduce(d.partials, (int)G, d.dcross, (K + 1) * S * S, prod);
  }
  {
    const double* sW = prod + K * S * S;
    double cn2 = 0.0;
    for (int jcl = 0; jcl < S; ++jcl) cn2 += sW[jcl * S + jcl];
    for (int i = tid; i < K; i += ORTH_NT) {
      const double* cr = prod + i * S * S;
      double acc = 0.0;
      for (int q = 0; q < S * S; ++q) acc += cr[q] * cr[q];
      exceed[i] = sqrt(acc) > d.orth_tol * sqrt(gk[i].trace) * sqrt(cn2);
    }
    csync();
    if (tid == 0) {
      int first = -1;
      for (int i = 0; i < K; ++i)
        if (exceed[i]) {
          first = i;
          break;
        }
      s_first = first;
      s_dec = first >= 0 ? 2 : 1;  // (the producer continues with the second pass, or stops)
      if (blockIdx.x == 0) {
        d.rec[RecLayout::kFirst] = first;
        d.rec[RecLayout::kReorth] = first >= 0 ? 1.0 : 0.0;
        d.st->reorth = first >= 0;
        d.st->zready = 0;
      }
    }
    csync();
  }
  orth_mark(d, 3);
  if (s_first >= 0) {
    // ---- pass 1: k rounds with t accumulated, then W of the new candidate.  Its round-0 products
    //      V_0^T cand[:,1:] are block 0 of the cross products just reduced (same candidate, same
    //      per-thread accumulation): no sweep and no barrier for them.
    for (int i = 0; i < K; ++i) {
      round(i, ((i + 1) & 1) ? d.dr1 : d.dr0, i + 1 == K, [&] { scalar(i, i == 0 ? -1 : (i & 1) ? d.dr1 : d.dr0, 1); });
      if (i + 1 < K) orth_gsync(&d.st->gbar, G);
    }
    cross_block(K, d.dwb);
    orth_gsync(&d.st->gbar, G);
    orth_mark(d, 4);
    // the candidate's raw Gram products for the least-squares stream (its snapshot: the next
    // block iteration reuses the partial regions)
    if (blockIdx.x == 0) {
      orth_reduce(d.partials, (int)G, d.dwb, S * S, tc);  // (ends with a barrier)
      if (tid < S * S) d.rec[d.rec_wraw + tid] = tc[tid];
    }
  } else {
    orth_mark(d, 4);
    if (blockIdx.x == 0 && tid < S * S) d.rec[d.rec_wraw + tid] = prod[K * S * S + tid];
  }
  orth_mark(d, 5);
  finish();
}

// dynamic shared memory of the block-iteration kernel without the ring
size_t orth_smem_base(int s, int k, int64_t P) {
  const size_t gramc = sizeof(double) * (2 + (size_t)s * s);  // GramC<s>
  return sizeof(double) * (64 + (size_t)orth_h_cap(k, s) + (size_t)orth_prod_cap(k, s)) + sizeof(Gram) +
         gramc * (size_t)k + sizeof(double) * (ORTH_NT / 32) * (s * s) + 16 +
         sizeof(double) * (size_t)std::max(1, std::min(s - 1, kOrthSmemCols)) * (size_t)P;
}
inline size_t orth_stage_bytes(int s) { return sizeof(double) * (size_t)s * ORTH_T; }
// ring stages that fit beside the largest launch of a cycle (k = m), at most kOrthMaxStages
int orth_stages(int s, int m, int64_t P) {
  const size_t b = orth_smem_base(s, m, P);
  if (b >= kOrthSmemCap) return 0;
  return (int)std::min<size_t>(kOrthMaxStages, (kOrthSmemCap - b) / orth_stage_bytes(s));
}
size_t orth_smem(int s, int k, int64_t P, int nst) { return orth_smem_base(s, k, P) + (size_t)nst * orth_stage_bytes(s); }

// ghost doubles of the level-by-level candidate powers (level j: e_j = s-1-j index rows of nx
// points on each side), or -1 when they do not apply (2D constant stencil only)
int64_t powers_ghost_doubles(const DevOp& op, int s, int64_t n) {
  if (op.kind != kStencilConst || op.dim != 2 || s < 2 || n >= (int64_t)1 << 30) return -1;
  // two regions used alternately: levels 0, 2, .. (e_0 = s-1 rows a side) and 1, 3, .. (e_1 = s-2)
  return s >= 3 ? 2 * (int64_t)(2 * s - 3) * op.nx : 0;
}

template <int S>
void run_orth(Ctx& c, const OrthDesc& d, int G, size_t smem) {
  ensure_smem(k_arn_step<S>, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = G;
  cfg.blockDim = ORTH_THREADS;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_arn_step<S>, d));
}

// r-norm after the cycle's residual update
__global__ void k_arn_rn(ArnState* st, const double* partials, int G, int dRR, double* out) {
  SKC_PDL_ENTRY();
  __shared__ double v[1];
  reduce_dots_dev(partials, G, dRR, 1, v);
  if (threadIdx.x == 0) {
    st->rn = sqrt(v[0]);
    *out = st->rn;
  }
}

// ---------------------------------------------------------------- standard GMRES pieces
struct GmState {
  int status;  // 0 running, 1 happy breakdown, 2 rho <= tol
  int halt;
  int step;
  int fin;     // back substitution: 1 ok, 2 rank-deficient
  double rn;
};

// cycle start: q_0 scale and HessenbergLsq(rn) (solvers.hpp:311-318)
__global__ void k_gm_start(GmState* st, double* coef, int cInv, void* lsq, int M) {
  SKC_PDL_ENTRY();
  if (threadIdx.x == 0) {
    st->status = 0;
    st->halt = 0;
    st->step = 0;
    st->fin = 0;
    coef[cInv] = 1.0 / st->rn;
    lsq_reset(lsq_view(lsq, M), st->rn);
  }
}

// inner step j's least-squares column (solvers.hpp:322-335): append H[:, j] (rows 0..j) to the
// Givens QR; rho <= tol ends the cycle (after a happy breakdown the column still counts)
__global__ void k_gm_lsq(GmState* st, double* col, int j, void* lsq, int M, double tol) {
  SKC_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  const bool happy = st->status == 1 && st->step == j;
  if (st->halt && !happy) return;
  const LsqView v = lsq_view(lsq, M);
  const double rho = lsq_append_serial(v, col);  // (rotated in place; col[j + 1] keeps the flag)
  if (!happy && rho <= tol) {
    st->status = 2;
    st->step = j;
    st->halt = 1;
  }
}

// end of the cycle: y (back substitution, solvers.hpp:336-343) into the update coefficients,
// zero past the appended columns; a rank failure leaves y = 0 (x untouched) and fin = 2
__global__ void k_gm_finish(GmState* st, void* lsq, int M, double* ycoef, int nterm) {
  SKC_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < nterm; ++i) ycoef[i] = 0.0;
  const LsqView v = lsq_view(lsq, M);
  if (!lsq_solve(v, false)) {
    st->fin = 2;
    return;
  }
  for (int i = 0; i < v.h->cols && i < nterm; ++i) ycoef[i] = v.y[i];
  st->fin = 1;
}

// col_i = q_i . w ; coefficient -col_i for the MGS update (solvers.hpp:94-97)
__global__ void k_gm_col(GmState* st, double* col, int i, double* coef, int cC, const double* partials, int G,
                         int d0) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    col[i] = v[0];
    coef[cC] = -v[0];
  }
}

// hsub = ||w||, happy-breakdown test against ||col|| (solvers.hpp:100-109)
__global__ void k_gm_sub(GmState* st, int j, double* col, double* coef, int cInv, const double* partials, int G,
                         int d0) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    const double hsub = sqrt(v[0]);
    col[j] = hsub;
    double acc = 0.0;
    for (int t = 0; t <= j; ++t) acc += col[t] * col[t];
    const bool happy = hsub <= 1e-14 * sqrt(acc);
    col[j + 1] = happy ? 1.0 : 0.0;  // flag stored past the column
    st->step = j;
    if (happy) {
      st->status = 1;
      st->halt = 1;
      return;
    }
    coef[cInv] = 1.0 / hsub;
  }
}

__global__ void k_gm_rn(GmState* st, const double* partials, int G, int d0) {
  SKC_PDL_ENTRY();
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) st->rn = sqrt(v[0]);
}

}  // namespace

// ============================================================================ standard GMRES
void gmres_device(Ctx& c, const Op& op, const double* f, double* x, uint64_t m64, double tol, uint64_t max_iterations,
                  Report& rep) {
  require(m64 >= 1, "gmres: restart length m must be at least 1");
  require(m64 <= 4096, "gmres: restart length above the device limit of 4096");
  const int m = (int)m64;
  const int64_t n = op.n;
  const size_t np = pad_n(n);
  const Geo g = make_geo_for(c, op);
  skc_op_counter& cnt = rep.op_counts;
  cnt.stored_vectors = m64 + 4;
  double* V = (double*)c.workspace("gm_vec", (size_t)(m + 4) * np * sizeof(double));
  double *r = V, *w = V + np, *ax = V + 2 * np, *Q = V + 3 * np;
  auto q = [&](int i) { return Q + (size_t)i * np; };
  const int cC = 0, cInv = 1, cM1 = 2, cY = 3, ncoef = 3 + m + 1;
  double* coef = (double*)c.workspace("gm_coef", ncoef * sizeof(double));
  double* partials = (double*)c.workspace("gm_partials", (size_t)2 * kPartialPitch * sizeof(double));
  const int rstride = m + 3;
  double* cols = (double*)c.workspace("gm_cols", (size_t)(m + 1) * rstride * sizeof(double));
  GmState* st = (GmState*)c.workspace("gm_state", sizeof(GmState));
  void* lsq = c.workspace("gm_lsq", lsq_bytes(m));
  const int* halt = &st->halt;
  {
    double hc[3] = {0.0, 0.0, -1.0};
    CK(cudaMemcpyAsync(coef, hc, sizeof hc, cudaMemcpyHostToDevice, c.stream));
    GmState h{};
    CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c.stream));
  }
  auto enqueue_residual = [&](bool x_zero) {
    LinBuilder lb;
    if (!x_zero) {
      launch_apply(c, op.d, x, ax, nullptr, nullptr);
      lb.add_out(r, f);
      lb.add_term(ax, 1u, cM1);
    } else {
      lb.add_out(r, f);
    }
    lb.add_dot(0, 0);
    lb.launch(c, g, coef, ncoef, partials, 0, nullptr, nullptr, "residual");
    launch_k(c, k_gm_rn, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), 0, 1), 0);
    ++c.launches;
  };
  const bool x_zero = device_is_zero(c, x, n);
  if (!x_zero) add(cnt, 0, 1, 1);
  enqueue_residual(x_zero);
  GmState hs;
  CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  double rn = hs.rn;
  cnt.termination_dots += 1;
  rep.history.push_back(rn);
  rep.op_history.push_back(cnt);
  std::vector<double> hcols((size_t)(m + 1) * rstride);
  while (rn > tol && rep.iterations < max_iterations) {
    const int steps = (int)std::min<uint64_t>((uint64_t)m, max_iterations - rep.iterations);
    CK(cudaMemsetAsync(cols, 0, (size_t)(m + 1) * rstride * sizeof(double), c.stream));
    launch_k(c, k_gm_start, 1, 32, 0, st, coef, cInv, lsq, m);
    ++c.launches;
    {
      LinBuilder lb;  // q_0 = r / ||r||
      lb.add_out(q(0), r, cInv);
      lb.launch(c, g, coef, ncoef, partials, 0, halt, nullptr, "scale");
    }
    for (int j = 1; j <= steps; ++j) {
      double* col = cols + (size_t)j * rstride;
      launch_apply(c, op.d, q(j - 1), w, halt, nullptr);
      launch_gram_list(c, g, {q(0)}, {w}, partials, 0, halt, nullptr, "gram");
      for (int i = 0; i < j; ++i) {
        launch_k(c, k_gm_col, 1, 256, 0, st, col, i, coef, cC, partials, c.reduce_point(partials, g.enc(), 0, 1), 0);
        ++c.launches;
        LinBuilder lb;  // w -= col_i q_i ; next dot
        lb.add_out(w, w);
        lb.add_term(q(i), 1u, cC);
        if (i + 1 < j) {
          lb.add_extra(q(i + 1));
          lb.add_dot(1, 0);
        } else {
          lb.add_dot(0, 0);
        }
        lb.launch(c, g, coef, ncoef, partials, 0, halt, nullptr, "mgs_update");
      }
      launch_k(c, k_gm_sub, 1, 256, 0, st, j, col, coef, cInv, partials, c.reduce_point(partials, g.enc(), 0, 1), 0);
      ++c.launches;
      LinBuilder lb;
      lb.add_out(q(j), w, cInv);
      lb.launch(c, g, coef, ncoef, partials, 0, halt, nullptr, "scale");
      launch_k(c, k_gm_lsq, 1, 32, 0, st, col, j, lsq, m, tol);
      ++c.launches;
    }
    // y, x += sum y_i q_i over the cycle's columns (zero past the appended ones), r = f - A x
    launch_k(c, k_gm_finish, 1, 32, 0, st, lsq, m, coef + cY, steps);
    ++c.launches;
    {
      LinBuilder lb;
      lb.add_out(x, x);
      for (int i = 0; i < steps; ++i) lb.add_term(q(i), 1u, cY + i);
      lb.launch(c, g, coef, ncoef, partials, 0, nullptr, nullptr, "x_update");
    }
    enqueue_residual(false);
    CK(cudaGetLastError());
    LsqHdr lh;
    CK(cudaMemcpyAsync(hcols.data(), cols, hcols.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&lh, lsq, sizeof lh, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    // replay the reference's inner loop on the device's decisions
    add(cnt, 0, 0, 1);  // q1 scaling
    bool happy = false;
    const int inner = lh.cols;
    for (int j = 1; j <= inner; ++j) {
      const bool hp = hcols[(size_t)j * rstride + j + 1] != 0.0;
      add(cnt, (uint64_t)j + 1, 1, (uint64_t)j + (hp ? 0 : 1));
      ++rep.iterations;
      if (hp) happy = true;
    }
    if (hs.fin != 1) {
      rep.breakdown = "hessenberg lsq: rank-deficient R diagonal at column " + std::to_string(lh.rank_col);
      break;
    }
    add(cnt, 0, 0, (uint64_t)inner);
    add(cnt, 0, 1, 1);
    ++rep.cycles;
    rn = hs.rn;
    cnt.termination_dots += 1;
    rep.history.push_back(rn);
    if (inner == m && !happy) rep.op_history.push_back(cnt);
    if (happy && rn > tol) {
      rep.breakdown = "happy breakdown but residual above threshold";
      break;
    }
  }
  rep.converged = rn <= tol;
  rep.final_residual = rep.history.back();
}

// ============================================================================ s-step Arnoldi engine
namespace {

// f(std::integral_constant<int, s>) for the block width s = 1..8
template <class F>
void dispatch_s(int s, F&& f) {
  switch (s) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    default: f(std::integral_constant<int, 8>{}); break;
  }
}

struct Engine {
  Ctx& c;
  const Op& op;
  int s, m;
  Geo g;
  size_t np;
  RecLayout rl;
  CoefLayout cl;
  DotLayout dl;
  double* V;  // (m+1) blocks of s columns
  double *z, *seed, *r, *ax;
  double* coef;
  double* partials;
  double* rec;
  double* scratch;
  double* rn_out;
  Gram* grams;
  ArnState* st;
  const int* halt;
  ArnLsqDesc lq{};      // least-squares state of the cycle (tol set per solve)
  const double* fvec = nullptr;  // the solve's right-hand side and iterate (device)
  double* xvec = nullptr;
  cudaEvent_t ev_step = nullptr, ev_lsq = nullptr;  // side-stream fork / join
  bool lsq_pending = false;
  bool zfused = false;  // the next block iteration's z and Scalar1 products are already computed
  // across GPUs the reorthogonalization decision is read back after the test (one stream sync
  // per block iteration), so a skipped second pass spends no collective and no halo exchange:
  // every rank reads the same decision (identical allgathered scalars)
  int host_reorth = -1;  // -1 unknown, else the last decision
  // the restart cycle as a CUDA graph: its launch sequence and arguments are identical for
  // every cycle of a solve (all control flow is device-side), so after one direct enqueue
  // (which also performs first-use allocations and kernel attribute setup) it is captured
  // once and replayed with a single launch per cycle
  cudaGraphExec_t cycle_exec = nullptr;
  uint64_t cycle_launches = 0;
  int cycles_enqueued = 0;

  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ~Engine() {
    if (cycle_exec) cudaGraphExecDestroy(cycle_exec);
    if (ev_step) cudaEventDestroy(ev_step);
    if (ev_lsq) cudaEventDestroy(ev_lsq);
  }

  // points per CTA of the on-chip orthogonalization (one CTA per SM), or 0 when it is off or
  // the candidate slices do not fit in shared memory
  // (spow: how the candidate powers run -- 2 row-aligned slices, 1 level by level on index
  // ranges, 0 per-level sweeps with grid barriers)
  int64_t orth_points(int* spow = nullptr) const {
    if (spow) *spow = 0;
    if (!c.orth || c.world() != 1 || g.grouped() || s < 2 || op.d.kind == kIlu0) return 0;
    const int G = mk_ctas();
    // (the geometry does not depend on the SKC_SPOW switch, only the powers' algorithm does)
    const int64_t gd = powers_ghost_doubles(op.d, s, op.n);
    auto ghosts_fit = [&](int64_t P) {
      return gd >= 0 && sizeof(double) * (size_t)gd <= (size_t)orth_stages(s, m, P) * orth_stage_bytes(s);
    };
    if (gd >= 0 && s >= 3 && op.d.nx % 2 == 0 && op.d.nx <= 2 * ORTH_NT) {
      // whole grid rows per CTA, for the row-wise candidate powers
      const int64_t P = (op.d.ny + G - 1) / G * op.d.nx;
      if (orth_stages(s, m, P) >= 2 && ghosts_fit(P)) {
        if (spow) *spow = c.spow ? 2 : 0;
        return P;
      }
    }
    const int64_t P = ((op.n + G - 1) / G + 1) & ~(int64_t)1;
    if (orth_stages(s, m, P) < 2) return 0;
    if (spow) *spow = c.spow && ghosts_fit(P) ? 1 : 0;
    return P;
  }

  // CTAs of the block-iteration kernel: one per SM, less the one SM left to the side stream's
  // least-squares kernels when they overlap the next block iteration
  int mk_ctas() const { return c.lsq_overlap ? c.sm_count - 1 : c.sm_count; }

  // block iteration k (z, Scalar1, seed, nu, candidate block, block MGS, reorthogonalization,
  // push) in one cooperative kernel
  void launch_step(int k, bool build_next) {
    OrthDesc d;
    std::memset(&d, 0, sizeof d);
    d.s = s;
    d.k = k;
    d.build_next = build_next ? 1 : 0;
    d.n = op.n;
    d.P = orth_points(&d.spow);
    d.op = op.d;
    d.vin = col(k - 1, s - 1);
    d.z = z;
    d.seed = seed;
    d.V = V;
    d.np = np;
    d.cand0 = col(k, 0);
    for (int j = 0; j < s; ++j) d.cand[j] = col(k, j);
    d.partials = partials;
    d.dz = dl.Z();
    d.dseed = dl.Seed();
    d.dr0 = dl.Dr(0);
    d.dr1 = dl.Dr(1);
    d.dcross = dl.Cross();
    d.dwb = dl.Wb();
    d.grams = grams;
    d.rec = recp(k);
    d.rec_push = recp(k - 1);
    d.rec_wraw = rl.wraw();
    d.rec_t = rl.t();
    d.rec_h = rl.h();
    d.st = st;
    d.orth_tol = 1e-8;
    d.reduced = scratch;  // (the per-phase kernels that use it do not run beside this one)
    static const int owner_dots = std::getenv("SKC_ORTH_OWNER_DOTS") ? std::atoi(std::getenv("SKC_ORTH_OWNER_DOTS")) : kOrthOwnerDots;
    d.owner_dots = owner_dots;
    static const bool trace = std::getenv("SKC_TRACE_ORTH") != nullptr;
    if (trace) d.trace = (unsigned long long*)c.workspace("orth_trace", 1024 * sizeof(unsigned long long));
    const int G = mk_ctas();
    d.nst = orth_stages(s, m, d.P);
    // (evict_first measured best on C2: 3913 vs 3845 s-steps/s unhinted, 3837 evict_last)
    static const int hint = std::getenv("SKC_ORTH_HINT") ? std::atoi(std::getenv("SKC_ORTH_HINT")) : 3;
    d.hint = hint;
    const size_t smem = orth_smem(s, k, d.P, d.nst);
    // algorithmic bytes, SURVEY 8(d) model (block-CGS-equivalent passes): a block step k < m
    // moves SpMV(2) + V^T z (ks+1) + seed (ks+2) + MPK (s+1) + V^T cand (ks+s) +
    // update/cross/Gram (ks+2s-1) = 4ks+4s+5 vectors, the last one (no build) 2ms+s+6.  The
    // implementation's block-MGS rounds and reorthogonalization pass are its own cost.
    const double ks = (double)k * s;
    const double bytes = 8.0 * (double)op.n * (build_next ? 4.0 * ks + 4.0 * s + 5.0 : 2.0 * ks + s + 6.0);
    Launch lh(c, "arn_step", bytes);
    switch (s) {
      case 2: run_orth<2>(c, d, G, smem); break;
      case 3: run_orth<3>(c, d, G, smem); break;
      case 4: run_orth<4>(c, d, G, smem); break;
      case 5: run_orth<5>(c, d, G, smem); break;
      case 6: run_orth<6>(c, d, G, smem); break;
      case 7: run_orth<7>(c, d, G, smem); break;
      default: run_orth<8>(c, d, G, smem); break;
    }
    lsq_fork(k, build_next);
    if (trace) {
      unsigned long long t[1024];
      CK(cudaMemcpyAsync(t, d.trace, sizeof t, cudaMemcpyDeviceToHost, c.stream));
      for (int ph = 1; ph <= 3; ++ph) {  // spread of the per-CTA phase completion times
        unsigned long long lo = ~0ull, hi = 0;
        int ilo = 0, ihi = 0;
        for (int b = 0; b < G; ++b) {
          const unsigned long long v = t[256 * ph + b];
          if (v < lo) lo = v, ilo = b;
          if (v > hi) hi = v, ihi = b;
        }
        std::fprintf(stderr, "[skew %s] %.1f us (first CTA %d, last CTA %d; CTA0 +%.1f)\n", ph == 1 ? "Zdots" : ph == 2 ? "seed" : "cross",
                     (hi - lo) * 1e-3, ilo, ihi, (t[256 * ph] - lo) * 1e-3);
      }
      c.sync();
      std::fprintf(stderr, "[step k=%d] z %.1f Zdots %.1f s1 %.1f seed %.1f s2 %.1f powers %.1f r0dots %.1f | rounds:", k,
                   (t[40] - t[39]) * 1e-3, (t[6] - t[40]) * 1e-3, (t[41] - t[6]) * 1e-3, (t[7] - t[41]) * 1e-3,
                   (t[42] - t[7]) * 1e-3, (t[43] - t[42]) * 1e-3, (t[0] - t[43]) * 1e-3);
      std::fprintf(stderr, " [lvl0 %.1f", (t[44] - t[42]) * 1e-3);
      for (int j = 1; j < s; ++j)
        std::fprintf(stderr, " sync %.1f lvl%d %.1f", (t[44 + 2 * j - 1] - t[44 + 2 * j - 2]) * 1e-3, j,
                     (t[44 + 2 * j] - t[44 + 2 * j - 1]) * 1e-3);
      std::fprintf(stderr, "]");
      for (int i = 0; i < k; ++i)
        std::fprintf(stderr, " (scal %.1f, upd %.1f, sync %.1f)", (t[8 + 3 * i] - (i ? t[7 + 3 * i] : t[0])) * 1e-3,
                     (t[9 + 3 * i] - t[8 + 3 * i]) * 1e-3, (t[10 + 3 * i] - t[9 + 3 * i]) * 1e-3);
      std::fprintf(stderr, " | znext %.1f cross %.1f sync %.1f check %.1f pass1 %.1f push %.1f us\n", (t[60] - t[7 + 3 * k]) * 1e-3, (t[1] - t[60]) * 1e-3,
                   (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3, (t[5] - t[4]) * 1e-3);
      std::fprintf(stderr, "[lsq k=%d] enter %.2f push/stage %.2f (push %.2f stage %.2f) gcols %.2f apply_l %.2f givens %.2f store %.2f (loop %.2f) us\n", k,
                   (t[70] - t[4]) * 1e-3, (t[71] - t[70]) * 1e-3, (t[76] - t[70]) * 1e-3, (t[77] - t[70]) * 1e-3,
                   (t[72] - t[71]) * 1e-3, (t[73] - t[72]) * 1e-3,
                   (t[74] - t[73]) * 1e-3, (t[75] - t[74]) * 1e-3, (t[78] - t[74]) * 1e-3);
    }
  }

  void enqueue_cycle_direct() {
    ctor(r, true);
    for (int k = 1; k <= m; ++k) advance(k, k < m);
    enqueue_finish(fvec, xvec);
  }

  // ctor(r) + the m block iterations of one restart cycle + its least-squares end, x update and
  // residual (the cycle's f and x are fixed for the solve: fvec, xvec)
  void enqueue_cycle() {
    static const bool graphs = [] {
      const char* e = std::getenv("SKC_GRAPH");
      return !e || std::atoi(e) != 0;
    }();
    // the per-phase trace reads its timestamps back after every block iteration, which a
    // stream capture cannot contain
    static const bool trace = std::getenv("SKC_TRACE_ORTH") != nullptr;
    const bool use_graph = graphs && !trace && c.world() == 1 && !c.profiling;
    if (!use_graph || cycles_enqueued++ == 0) return enqueue_cycle_direct();
    if (!cycle_exec) {
      const uint64_t l0 = c.launches;
      CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_cycle_direct();
      } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(c.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      cudaGraph_t graph = nullptr;
      CK(cudaStreamEndCapture(c.stream, &graph));
      const cudaError_t e = cudaGraphInstantiate(&cycle_exec, graph, 0);
      cudaGraphDestroy(graph);
      CK(e);
      cycle_launches = c.launches - l0;
      c.launches = l0;
    }
    CK(cudaGraphLaunch(cycle_exec, c.stream));
    c.launches += cycle_launches;
  }

  Engine(Ctx& ctx, const Op& o, int s_, int m_, bool fixed = false)
      : c(ctx), op(o), s(s_), m(m_), rl{s_, m_}, cl{s_, m_}, dl{s_, m_} {
    g = make_geo_for(c, op);
    np = pad_n(op.n);
    const size_t nvec = (size_t)(m + 1) * s + 4;
    V = (double*)c.workspace("arn_vec", nvec * np * sizeof(double));
    z = V + (size_t)(m + 1) * s * np;
    seed = z + np;
    r = seed + np;
    ax = r + np;
    coef = (double*)c.workspace("arn_coef", (size_t)cl.size() * sizeof(double));
    partials = (double*)c.workspace("arn_partials", (size_t)dl.size() * kPartialPitch * sizeof(double));
    rec = (double*)c.workspace("arn_rec", (size_t)(m + 1) * rl.size() * sizeof(double));
    scratch = (double*)c.workspace("arn_scratch", (size_t)(m * s * s + s * s + m * s + 8) * sizeof(double));
    rn_out = (double*)c.workspace("arn_rn", 8 * sizeof(double));
    grams = (Gram*)c.workspace("arn_grams", (size_t)(m + 1) * sizeof(Gram));
    st = (ArnState*)c.workspace("arn_state", sizeof(ArnState));
    halt = &st->halt;
    lq.s = s;
    lq.m = m;
    lq.GL = arn_lsq_ld(s, m);
    lq.lsq_on = 1;
    lq.tol = 0.0;
    lq.gcols = (double*)c.workspace("arn_gcols", (size_t)m * s * lq.GL * sizeof(double));
    lq.lblk = (double*)c.workspace("arn_lblk", (size_t)(m + 1) * s * s * sizeof(double));
    lq.lsq = c.workspace("arn_lsq", lsq_bytes(m * s));
    lq.rec = rec;
    lq.recsz = rl.size();
    lq.rec_t = rl.t();
    lq.rec_h = rl.h();
    lq.rec_wraw = rl.wraw();
    lq.st = st;
    lq.grams = grams;
    std::vector<double> hc(cl.size(), 0.0);
    hc[cl.M1()] = -1.0;
    CK(cudaMemcpyAsync(coef, hc.data(), hc.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    CK(cudaEventCreateWithFlags(&ev_step, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_lsq, cudaEventDisableTiming));
    ArnState h{};
    h.fixed = fixed ? 1 : 0;
    CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c.stream));
  }

  double* col(int block, int j) const { return V + ((size_t)block * s + j) * np; }
  double* recp(int k) const { return rec + (size_t)k * rl.size(); }

  // [v, A v, .., A^{s-1} v] of v = src * coef[Inv] into block slot b (krylov_block,
  // block.hpp:59-67).  Stencil operators use the matrix-powers kernel (one sweep, depth s-1,
  // chained in 3D past depth 3); when `dots` is set and a single sweep suffices, the first
  // block-MGS products V_0^T cand[:,1:] are fused into it.  Returns the partial count of the
  // fused products, or 0 when they were not computed.
  int krylov_into(int b, const double* src, bool dots = false) {
    const int J = s - 1, maxj = powers_depth(c, op.d);
    if (J >= 1 && maxj >= 1) {
      int done = 0;
      const double* from = src;
      const double* sc = coef + cl.Inv();
      int Gd = 0;
      while (done < J) {
        const int d = std::min(J - done, maxj);
        double* outs[kMaxS + 1];
        for (int j = 0; j <= d; ++j) outs[j] = col(b, done + j);
        if (done > 0) outs[0] = nullptr;  // already written by the previous sweep
        const double* X[kMaxS];
        // (on one GPU the 3D powers take the one-sweep kernel, which fuses no products)
        const bool fuse = dots && done == 0 && d == J && J <= kMpkMaxDotDepth && !g.grouped() &&
                          !(op.d.dim == 3 && c.world() == 1);
        for (int l = 0; l < s; ++l) X[l] = col(0, l);
        const int G0 = launch_mpk(c, op.d, from, sc, outs, d, fuse ? s : 0, X, 1, partials, dl.D(), halt, nullptr);
        if (fuse) Gd = G0;
        from = col(b, done + d);
        sc = nullptr;
        done += d;
      }
      return Gd;
    }
    LinBuilder lb;
    lb.add_out(col(b, 0), src, cl.Inv());
    lb.launch(c, g, coef, cl.size(), partials, 0, halt, nullptr, "scale");
    for (int j = 1; j < s; ++j) launch_apply(c, op.d, col(b, j - 1), col(b, j), halt, nullptr);
    return 0;
  }

  // y = A x (skipped unless *cond when given)
  void apply(const double* x, double* y, const int* cond = nullptr) { launch_apply(c, op.d, x, y, halt, cond); }

  void gram_self_into(int b, int dW, const int* cond, const char* name = "gram_w") {
    std::vector<const double*> B;
    for (int j = 0; j < s; ++j) B.push_back(col(b, j));
    launch_gram_list(c, g, B, B, partials, dW, halt, cond, name);
  }

  // SStepArnoldi ctor on device vector v (use_rn: its norm is st->rn)
  void ctor(const double* v, bool use_rn) {
    zfused = false;
    host_reorth = -1;
    CK(cudaMemsetAsync(rec, 0, (size_t)(m + 1) * rl.size() * sizeof(double), c.stream));
    if (!use_rn) launch_gram_list(c, g, {v}, {v}, partials, dl.RR(), nullptr, nullptr, "gram");
    const int Gc = use_rn ? g.enc() : c.reduce_point(partials, g.enc(), dl.RR(), 1);
    launch_k(c, k_arn_ctor, 1, 256, 0, st, use_rn ? 1 : 0, partials, Gc, dl.RR(), recp(0), coef, cl.Inv());
    ++c.launches;
    krylov_into(0, v);
    gram_self_into(0, dl.Wa(), nullptr);
    const int Gw = c.reduce_point(partials, g.enc(), dl.Wa(), s * s);
    dispatch_s(s, [&](auto S_) {
      constexpr int S = decltype(S_)::value;
      launch_k(c, k_arn_ctor_push<S>, 1, 256, 0, lq, (const double*)partials, Gw, dl.Wa());
    });
    ++c.launches;
    CK(cudaGetLastError());
  }

  // block step k's least squares (k_arn_lsq) on the side stream, after the block step's kernels
  // (the next block step does not wait for it; lsq_join does)
  void lsq_fork(int k, bool build_next) {
    int cap = arn_lsq_scratch(s, m);
    if ((size_t)(cap + arn_lsq_prev(s, m)) * sizeof(double) <= 200 * 1024) cap += arn_lsq_prev(s, m);
    const size_t smem = sizeof(double) * (size_t)cap;
    cudaStream_t a = c.stream;
    if (c.lsq_overlap) {
      a = c.aux();
      CK(cudaEventRecord(ev_step, c.stream));
      CK(cudaStreamWaitEvent(a, ev_step, 0));
      lsq_pending = true;
    }
    dispatch_s(s, [&](auto S_) {
      constexpr int S = decltype(S_)::value;
      ensure_smem(k_arn_lsq<S>, smem);
      k_arn_lsq<S><<<1, 256, smem, a>>>(lq, k, build_next ? 1 : 0, cap);
    });
    CK(cudaGetLastError());
    ++c.launches;
  }
  void lsq_join() {
    if (!lsq_pending) return;
    CK(cudaEventRecord(ev_lsq, c.aux()));
    CK(cudaStreamWaitEvent(c.stream, ev_lsq, 0));
    lsq_pending = false;
  }

  // end of the cycle on the device: y (k_arn_finish), x += V y over the m blocks (zero
  // coefficients past the appended columns), r = f - A x and ||r|| (st->rn, rn_out)
  void enqueue_finish(const double* f, double* x) {
    lsq_join();
    const size_t fsm = sizeof(double) * fin_smem_doubles(m * s);
    ensure_smem(k_arn_finish, fsm);
    launch_k(c, k_arn_finish, 1, 256, fsm, lq, coef + cl.Y());
    ++c.launches;
    LinBuilder lb;
    lb.add_out(x, x);
    for (int bi = 0; bi < m; ++bi)
      for (int lc = 0; lc < s; ++lc) lb.add_term(col(bi, lc), 1u, cl.Y() + bi * s + lc);
    lb.launch(c, g, coef, cl.size(), partials, 0, nullptr, nullptr, "x_update");
    enqueue_residual(f, x, false);
  }

  // r = f - A x (or f when x is known zero), ||r|| -> st->rn and rn_out
  void enqueue_residual(const double* f, const double* x, bool x_zero) {
    LinBuilder lb;
    if (!x_zero) {
      launch_apply(c, op.d, x, ax, nullptr, nullptr);
      lb.add_out(r, f);
      lb.add_term(ax, 1u, cl.M1());
    } else {
      lb.add_out(r, f);
    }
    lb.add_dot(0, 0);
    lb.launch(c, g, coef, cl.size(), partials, dl.RR(), nullptr, nullptr, "residual");
    launch_k(c, k_arn_rn, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), dl.RR(), 1), dl.RR(), rn_out);
    ++c.launches;
  }

  // SStepArnoldi::advance for block iteration k (1-based), sstep.hpp:297-379
  void advance(int k, bool build_next) {
    if (orth_points() > 0) {  // the whole block iteration on chip
      launch_step(k, build_next);
      return;
    }
    double* rk = recp(k);
    // z = A v_k^s ; Scalar1 dots V_i^T z and ||z||^2.  After a block iteration that fused them
    // into its cross-product pass (zfused) they are already in place, unless that iteration's
    // reorthogonalization pass changed the block: then (device flag) they are recomputed.
    const int* zcond = zfused ? &st->reorth : nullptr;
    const bool zskip = zfused && host_reorth == 0;  // (known on the host: nothing to redo)
    zfused = false;
    if (!zskip) {
      apply(col(k - 1, s - 1), z, zcond);
      std::vector<const double*> L;
      for (int i = 0; i < k; ++i)
        for (int l = 0; l < s; ++l) L.push_back(col(i, l));
      L.push_back(z);
      launch_gram_list(c, g, L, {z}, partials, dl.Z(), halt, zcond, zcond ? "gram_z_redo" : "gram_z");
    }
    launch_k(c, k_arn_s1, 1, 256, 0, st, grams, k, rk, coef, partials, c.reduce_point(partials, g.enc(), dl.Z(), k * s + 1), dl.Z(), s, cl.H(), scratch);
    ++c.launches;
    // seed = z - sum_i V_i h_i ; ||seed||^2
    {
      LinBuilder lb;
      lb.add_out(seed, z);
      for (int i = 0; i < k; ++i)
        for (int l = 0; l < s; ++l) lb.add_term(col(i, l), 1u, cl.H() + i * s + l);
      lb.add_dot(0, 0);
      lb.launch(c, g, coef, cl.size(), partials, dl.Seed(), halt, nullptr, "seed_update");
    }
    launch_k(c, k_arn_s2, 1, 256, 0, st, k, rk, coef, partials, c.reduce_point(partials, g.enc(), dl.Seed(), 1), dl.Seed(), cl.Inv());
    ++c.launches;
    // candidate block [v, .., A^{s-1} v] of the normalized seed (also on the last block)
    const int cb = k;  // block slot k (slot m is scratch when k == m)
    const int Gfused = krylov_into(cb, seed, build_next && s > 1);
    if (!build_next) {
      lsq_fork(k, false);
      CK(cudaGetLastError());
      return;
    }
    double* tk = rk + rl.t();
    bool wb_needed = true;  // the reorthogonalized W region must be made global for the push
    if (s > 1) {
      int Gcross = g.enc();
      for (int pass = 0; pass < 2; ++pass) {
        // Across ranks the second pass is enqueued under the device flag like on one GPU: its
        // kernels skip when the test did not fire, its collectives run (on stale, unused values)
        // so every rank issues the same sequence without a host round trip.  SKC_REORTH_SYNC=1
        // reads the decision back instead (one stream sync per block iteration, no idle collectives).
        if (pass == 1 && c.world() > 1 && c.reorth_host_sync) {
          host_reorth = read_state().reorth;
          if (!host_reorth) {
            wb_needed = false;
            break;
          }
        }
        const int* cond = pass ? &st->reorth : nullptr;
        std::vector<const double*> Cr;
        for (int jc = 1; jc < s; ++jc) Cr.push_back(col(cb, jc));
        const bool have = pass == 0 && Gfused > 0;  // products already fused into the powers sweep
        // (the second pass' round-0 products V_0^T cand[:,1:] are block 0 of the cross products)
        if (!have && pass == 0) {
          std::vector<const double*> L;
          for (int l = 0; l < s; ++l) L.push_back(col(0, l));
          launch_gram_list(c, g, L, Cr, partials, dl.D(), halt, cond, pass ? "gram_mgs_reorth" : "gram_mgs");
        }
        for (int i = 0; i < k; ++i) {
          const int Gi = (i == 0 && have) ? Gfused : g.enc();
          // Scalar2 against block i (sstep.hpp:338-353) runs in the update kernel's prologue:
          // t = W_i^{-1} V_i^T cand[:,1:], recorded at block i of this iteration's T area
          const bool from_cross = pass == 1 && i == 0;
          const MgsScalar sc{partials,
                             from_cross ? Gcross : c.reduce_point(partials, Gi, dl.Dr(i), s * (s - 1)),
                             from_cross ? dl.Cross() : dl.Dr(i),
                             grams + i,
                             tk + i * s * s,
                             pass,
                             from_cross ? 1 : 0};
          // cand[:,jc] -= sum_l t(l,jc-1) V_i[:,l]  (+ products with V_{i+1})
          const double* Vi[kMaxS];
          const double* Vn[kMaxS];
          double* cd[kMaxS];
          for (int l = 0; l < s; ++l) {
            Vi[l] = col(i, l);
            Vn[l] = i + 1 < k ? col(i + 1, l) : nullptr;
            cd[l] = col(cb, l);
          }
          launch_mgs(c, g, s, Vi, cd, i + 1 < k ? Vn : nullptr, sc, partials, dl.Dr(i + 1), halt, cond,
                     pass ? "mgs_update_reorth" : "mgs_update");
        }
        if (pass == 0) {
          // reorthogonalization test and the candidate's Gram matrix in one pass over cand:
          // [V_0..V_{k-1}, cand]^T cand -> cross blocks, then W at Cross + k s^2.  When the
          // next block iteration follows, its z = A cand[:,s-1] is formed now and its Scalar1
          // products [V_0..V_{k-1}, cand, z]^T z ride in the same pass (Z region).
          std::vector<const double*> L, R;
          std::vector<GramCol> cols;
          for (int i = 0; i < k; ++i)
            for (int l = 0; l < s; ++l) L.push_back(col(i, l));
          for (int jc = 0; jc < s; ++jc) {
            L.push_back(col(cb, jc));
            R.push_back(col(cb, jc));
            cols.push_back({dl.Cross() + jc, s, (k + 1) * s});
          }
          if (s + 1 <= GR_MAXR) {
            apply(col(cb, s - 1), z);
            L.push_back(z);
            R.push_back(z);
            cols.push_back({dl.Z(), 1, (k + 1) * s + 1});
            zfused = true;
          }
          launch_gram_map(c, g, L, R, cols, partials, halt, nullptr, "gram_cross");
          Gcross = c.reduce_point(partials, g.enc(), dl.Cross(), k * s * s + s * s);
          launch_k(c, k_arn_check, 1, 256, 0, st, grams, k, rk, partials, Gcross, dl.Cross(), dl.Cross() + k * s * s, s, 1e-8, scratch);
          ++c.launches;
        } else {
          gram_self_into(cb, dl.Wb(), cond, "gram_w_reorth");
        }
      }
    }
    const int dWa = s > 1 ? dl.Cross() + k * s * s : dl.Wa();
    if (s == 1) gram_self_into(cb, dl.Wa(), nullptr);
    // the push reads W from the reorthogonalized region when the device flag says so: make
    // both regions global (the unused one is stale but harmless)
    // (for s > 1 the dWa region was already made global together with the cross products)
    const int Gw = s > 1 ? (wb_needed ? c.reduce_point(partials, g.enc(), dl.Wb(), s * s) : c.world())
                         : c.reduce_point(partials, g.enc(), dWa, s * s);
    launch_k(c, k_arn_push, 1, 256, 0, st, grams, cb, rk, rl.wraw(), (const double*)partials, Gw, dWa, dl.Wb(), s);
    ++c.launches;
    lsq_fork(k, true);
    CK(cudaGetLastError());
  }

  ArnState read_state() {
    ArnState h;
    CK(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h;
  }
};

// Host view of the cycle's device records: the op counts of each advance (sstep.hpp:297-379)
// and the recorded Gram matrices -- bookkeeping only, no arithmetic on the solve's numbers.
struct HostArn {
  int s, m;
  RecLayout rl;
  std::vector<double> recs;  // copied records

  const double* rec(int k) const { return recs.data() + (size_t)k * rl.size(); }

  std::vector<double> W(int k) const {
    const double* r = rec(k);
    return std::vector<double>(r + RecLayout::kW, r + RecLayout::kW + s * s);
  }

  // op counts of advance(k, build_next); stage: 0 = complete, 1 = invariant return,
  // 2 = push_block threw (counts through the Gram products)
  mutable uint64_t reorth_passes = 0;  // diagnostics (SKC_TRACE)
  void count_advance(skc_op_counter& c, int k, bool build_next, int stage) const {
    const uint64_t S = s;
    add(c, (uint64_t)k * S + 1, 1, (uint64_t)k * S);  // z, Scalar1, seed, nu
    if (stage == 1) return;
    add(c, 0, S - 1, 1);  // scale + candidate block
    if (!build_next) return;
    if (s > 1) {
      add(c, (uint64_t)k * S * (S - 1), 0, (uint64_t)k * S * (S - 1));
      const double* r = rec(k);
      const int first = (int)r[RecLayout::kFirst];
      const bool reorth = r[RecLayout::kReorth] != 0.0;
      if (reorth) ++reorth_passes;
      add(c, S + S * S * (uint64_t)(reorth ? first + 1 : k), 0, 0);
      if (reorth) add(c, (uint64_t)k * S * (S - 1), 0, (uint64_t)k * S * (S - 1));
    }
    add(c, S * (S + 1) / 2, 0, 0);  // push_block Gram
  }
};

}  // namespace

// ============================================================================ s-GMRES
void sgmres_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep) {
  require(cfg.m >= 1, "s-gmres: m must be at least 1");
  validate_block_size(cfg, rep);
  if (cfg.s == 1) {  // sstep.hpp:498-508
    Report sub;
    gmres_device(c, op, f, x, cfg.m, cfg.tol, cfg.max_iterations, sub);
    sub.notes = rep.notes;
    rep = std::move(sub);
    return;
  }
  require(cfg.m <= 64, "s-gmres: m above the device limit of 64 blocks");
  const int s = (int)cfg.s, m = (int)cfg.m;
  skc_op_counter& cnt = rep.op_counts;
  cnt.stored_vectors = (uint64_t)(m + 2) * s + 2;
  Engine E(c, op, s, m, cfg.fixed_steps);
  E.lq.tol = cfg.tol;
  E.fvec = f;
  E.xvec = x;
  HostArn H{s, m, E.rl, {}};
  H.recs.resize((size_t)(m + 1) * E.rl.size());

  auto read_rn = [&]() {
    double h;
    CK(cudaMemcpyAsync(&h, E.rn_out, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h;
  };
  const bool x_zero = device_is_zero(c, x, op.n);
  if (!x_zero) add(cnt, 0, 1, 1);
  E.enqueue_residual(f, x, x_zero);
  double rn = read_rn();
  cnt.termination_dots += 1;
  rep.history.push_back(rn);
  rep.op_history.push_back(cnt);

  // sstep.hpp:518-543
  auto run_fallback = [&]() -> bool {
    Report sub;
    gmres_device(c, op, f, x, (uint64_t)s * m, cfg.tol, (uint64_t)s * m, sub);
    rep.iterations += sub.iterations;
    rep.cycles += sub.cycles;
    ++rep.fallback_cycles;
    cnt.dotprods += sub.op_counts.dotprods;
    cnt.matvecs += sub.op_counts.matvecs;
    cnt.vec_updates += sub.op_counts.vec_updates;
    cnt.termination_dots += sub.op_counts.termination_dots;
    for (size_t i = 1; i < sub.history.size(); ++i) rep.history.push_back(sub.history[i]);
    add(cnt, 0, 1, 1);
    E.enqueue_residual(f, x, false);
    rn = read_rn();
    cnt.termination_dots += 1;
    rep.op_history.push_back(cnt);
    return rn <= cfg.tol;
  };

  while (rn > cfg.tol && rep.iterations < cfg.max_iterations) {
    bool collapsed = false, exhausted = false;
    std::string collapse_msg;
    int blocks_done = 0;
    // ---- the whole cycle on the device (one graph), then one read-back
    E.enqueue_cycle();
    ArnState hs;
    LsqHdr lh;
    double cycle_rn = 0.0;
    CK(cudaMemcpyAsync(&hs, E.st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&lh, E.lq.lsq, sizeof lh, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&cycle_rn, E.rn_out, sizeof cycle_rn, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(H.recs.data(), E.rec, H.recs.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    // ---- replay the reference's cycle loop (sstep.hpp:546-654) on the device's decisions
    if (hs.status == kArnCtorZero) fail(SKC_EINVAL, "s-arnoldi: start vector is zero");
    add(cnt, (uint64_t)s * (s + 1) / 2, (uint64_t)s - 1, 1);  // ctor: scale, krylov_block, push
    if (hs.status == kArnCtorCollapse) {
      collapse_msg = gram_message((int)H.rec(0)[RecLayout::kSing], H.rec(0)[RecLayout::kRatio]);
      if (!run_fallback()) {
        if (rep.iterations >= cfg.max_iterations) break;
        continue;
      }
      break;
    }
    // (cholesky_upper of block 0 escapes sgmres_solve in the reference, sstep.hpp:563)
    if (hs.status == kArnCtorChol) fail(SKC_EBREAKDOWN, "cholesky: matrix not positive definite");
    for (int k = 1; k <= m; ++k) {
      // (the least-squares stream's verdict on the block steps; the constructor's is hs.status)
      const bool stopped_here = hs.lstatus != kArnRunning && hs.lblock == k;
      const bool invariant = stopped_here && hs.lstatus == kArnInvariant;
      H.count_advance(cnt, k, k < m, invariant ? 1 : 0);
      if (stopped_here && hs.lstatus == kArnPushCollapse) {
        collapsed = true;
        collapse_msg = gram_message((int)H.rec(k)[RecLayout::kSing], H.rec(k)[RecLayout::kRatio]);
        break;
      }
      if (stopped_here && hs.lstatus == kArnCholCollapse) {
        collapsed = true;
        collapse_msg = "cholesky: matrix not positive definite";
        break;
      }
      const double rho = H.rec(k)[RecLayout::kRho];
      rep.block_rho.push_back(rho);
      rep.iterations += s;
      blocks_done = k;
      if (invariant) {
        exhausted = true;
        break;
      }
      if (rho <= cfg.tol) break;  // (the device stopped the cycle here: kArnEarly)
    }
    if (hs.fin == kFinFallback) {  // collapsed, residual estimate above tol: x untouched
      if (!run_fallback()) {
        if (rep.iterations >= cfg.max_iterations) {
          rep.breakdown = "basis collapse (" + collapse_msg + ")";
          break;
        }
        continue;
      }
      break;
    }
    if (hs.fin == kFinLsqFail) {  // x untouched (y = 0)
      rep.breakdown = "hessenberg lsq: rank-deficient R diagonal at column " + std::to_string(lh.rank_col);
      break;
    }
    // x += sum_bi sum_lc y V ; r = f - A x (sstep.hpp:622-633), done on the device
    add(cnt, 0, 0, (uint64_t)blocks_done * s);
    add(cnt, 0, 1, 1);
    ++rep.cycles;
    rn = cycle_rn;
    cnt.termination_dots += 1;
    rep.history.push_back(rn);
    if (blocks_done == m && !exhausted && !collapsed) rep.op_history.push_back(cnt);
    if (rn <= cfg.tol) break;
    if (collapsed) {
      if (!run_fallback() && rep.iterations >= cfg.max_iterations) {
        rep.breakdown = "basis collapse (" + collapse_msg + ")";
        break;
      }
      if (rn <= cfg.tol) break;
      continue;
    }
    if (exhausted) {
      rep.breakdown = "invariant subspace reached with residual above threshold";
      break;
    }
  }
  rep.converged = rn <= cfg.tol;
  if (std::getenv("SKC_TRACE"))
    std::fprintf(stderr, "[skc] s-gmres: %llu cycles, %llu reorthogonalization passes\n",
                 (unsigned long long)rep.cycles, (unsigned long long)H.reorth_passes);
  rep.final_residual = rep.history.back();
}

// ============================================================================ sarnoldi
void sarnoldi_device(Ctx& c, const Op& op, const double* v1, uint64_t s64, uint64_t m64, BasisOut& out) {
  require(s64 >= 1, "sarnoldi: s must be at least 1");
  require(m64 >= 1, "sarnoldi: m_blocks must be at least 1");
  require(s64 * m64 <= (uint64_t)op.n, "sarnoldi: s * m_blocks exceeds the dimension");
  require(s64 <= (uint64_t)kMaxS, "sarnoldi: s above the supported block width 8");
  require(m64 <= 64, "sarnoldi: m_blocks above the device limit of 64");
  const int s = (int)s64, m = (int)m64;
  Engine E(c, op, s, m);
  E.lq.lsq_on = 0;  // the basis and its Hessenberg columns only
  HostArn H{s, m, E.rl, {}};
  H.recs.resize((size_t)(m + 1) * E.rl.size());
  E.ctor(v1, false);
  for (int k = 1; k <= m; ++k) E.advance(k, k < m);
  E.lsq_join();
  ArnState hs = E.read_state();
  CK(cudaMemcpy(H.recs.data(), E.rec, H.recs.size() * sizeof(double), cudaMemcpyDeviceToHost));
  if (hs.status == kArnCtorZero) fail(SKC_EINVAL, "s-arnoldi: start vector is zero");
  if (hs.status == kArnCtorCollapse)
    fail(SKC_EBREAKDOWN, gram_message((int)H.rec(0)[RecLayout::kSing], H.rec(0)[RecLayout::kRatio]));
  skc_op_counter& cnt = out.counter;
  add(cnt, (uint64_t)s * (s + 1) / 2, (uint64_t)s - 1, 1);
  for (int k = 1; k <= m; ++k) {
    const bool stopped_here = hs.status != kArnRunning && hs.block == k;
    if (stopped_here && hs.status == kArnPushCollapse) {
      H.count_advance(cnt, k, k < m, 0);
      fail(SKC_EBREAKDOWN, gram_message((int)H.rec(k)[RecLayout::kSing], H.rec(k)[RecLayout::kRatio]));
    }
    if (stopped_here && hs.status == kArnInvariant) {
      H.count_advance(cnt, k, k < m, 1);
      fail(SKC_EBREAKDOWN, "sarnoldi: invariant subspace at block " + std::to_string(k));
    }
    H.count_advance(cnt, k, k < m, 0);
  }
  const size_t n = (size_t)op.n;
  out.blocks.assign((size_t)m * s * n, 0.0);
  for (int b = 0; b < m; ++b)
    for (int j = 0; j < s; ++j)
      CK(cudaMemcpy(out.blocks.data() + ((size_t)b * s + j) * n, E.col(b, j), n * sizeof(double),
                    cudaMemcpyDeviceToHost));
  out.grams.assign((size_t)m * s * s, 0.0);
  for (int b = 0; b < m; ++b) {
    const auto w = H.W(b);
    std::copy(w.begin(), w.end(), out.grams.begin() + (size_t)b * s * s);
  }
  // the block Hessenberg matrix (hessenberg(), sstep.hpp:383-389) from the device's columns
  const size_t rows = (size_t)(m + 1) * s, cols = (size_t)m * s, GL = (size_t)E.lq.GL;
  std::vector<double> gc(cols * GL);
  CK(cudaMemcpy(gc.data(), E.lq.gcols, gc.size() * sizeof(double), cudaMemcpyDeviceToHost));
  out.hess.assign(rows * cols, 0.0);
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < j + 2 && i < rows; ++i) out.hess[i * cols + j] = gc[j * GL + i];
  out.seed.assign(n, 0.0);
  CK(cudaMemcpy(out.seed.data(), E.col(m, 0), n * sizeof(double), cudaMemcpyDeviceToHost));
  out.seed_norm = H.rec(m)[RecLayout::kNu];
}

}  // namespace skc
