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
  int pad;
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
// One cooperative kernel for the whole block-MGS stage of a block iteration (sstep.hpp:331-379)
// when the candidate columns cand[:,1:] of every CTA's point slice fit in its shared memory:
// one CTA per SM owns points [b*P, (b+1)*P) and keeps its slice of cand[:,1:] on chip for
//   pass 0: k rounds  (Scalar2 solve in every CTA, cand -= V_i t, products V_{i+1}^T cand),
//   the cross products [V_0..V_{k-1}, cand]^T cand and the reorthogonalization test,
//   pass 1 (only when the test fires): V_0^T cand, k more rounds (t accumulated), W = cand^T cand,
// separated by grid-wide barriers; cand[:,1:] is written back once at the end.  Only the basis
// blocks stream from memory.  Every CTA reduces the per-CTA partials in the same fixed order,
// so all CTAs take identical coefficients and the same reorthogonalization decision; CTA 0
// writes the records and the device flags.
constexpr int ORTH_NT = 512;
// points per thread per iteration, all their loads issued first (Scalar1 products, seed):
// 8 x s loads of 8 bytes per thread ~ the unified L1 left beside the candidate slice (4 -> 8:
// C2 3848 -> 3909 s-steps/s)
constexpr int ORTH_UC = 8;
constexpr size_t kOrthSmemCap = 220 * 1024;
// candidate columns kept in shared memory (the rest in their basis slots): shared memory is
// carved out of the unified L1, whose remaining capacity bounds the loads in flight per SM
// (C2, s = 4: 3 columns on chip 3697 s-steps/s, 2 columns 3750, 1 column 3635)
#ifndef SKC_ORTH_SMEM_COLS
#define SKC_ORTH_SMEM_COLS 2
#endif
constexpr int kOrthSmemCols = SKC_ORTH_SMEM_COLS;
#ifndef SKC_HOIST
#define SKC_HOIST 0
#endif
#ifndef SKC_UU4
#define SKC_UU4 3
#endif  // <= the 226 KB dynamic limit set at launch
// reduced-product capacity: the cross test needs (k+1) s^2, a round s(s-1); even count keeps
// the Gram copy 16-byte aligned
__host__ __device__ inline int orth_prod_cap(int k, int s) { return ((k + 1) * s * s + 1) & ~1; }
constexpr int kStepH = 64 * kMaxS;  // -h coefficients of Scalar1 (k s <= 512)

struct OrthDesc {
  int s, k, build_next;
  int zfuse;              // form the next iteration's z and Scalar1 products in the cross pass
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
  // row-streamed candidate powers (2D constant stencil, s <= 4): per-CTA ghost-row buffers of
  // levels 1 and 2 (g1 + g2 doubles per CTA at ghosts); spow 0 = per-level sweeps with grid
  // barriers.  The buffers are in (L2-resident) global memory: shared memory beyond the
  // candidate slice would shrink the L1 share of the unified L1/shared array, whose capacity
  // bounds the loads in flight per SM for every streaming phase (measured: -14% on C2)
  int spow, g1, g2;
  double* ghosts;
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

// streamed basis loads: L2 only (no L1 allocation), so the number of loads in flight per SM is
// not bounded by the L1 capacity left beside the candidate slice in the unified L1/shared memory
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// fixed-order CTA reduction of K per-thread accumulators into partial column blockIdx.x
template <int K>
__device__ __forceinline__ void orth_store(const double (&acc)[K], double* red, double* partials, int d0) {
  constexpr int NW = ORTH_NT / 32;
  const int warp = threadIdx.x >> 5;
  warp_sums(acc, red + warp * K);
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w * K + threadIdx.x];
    partials[(int64_t)(d0 + threadIdx.x) * kPartialPitch + blockIdx.x] = s;
  }
  __syncthreads();
}

// as orth_store, products q < K1 to partials d0 + q and the rest to d1 + (q - K1)
template <int K, int K1>
__device__ __forceinline__ void orth_store2(const double (&acc)[K], double* red, double* partials, int d0, int d1) {
  constexpr int NW = ORTH_NT / 32;
  const int warp = threadIdx.x >> 5;
  warp_sums(acc, red + warp * K);
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w * K + threadIdx.x];
    const int q = threadIdx.x;
    partials[(int64_t)(q < K1 ? d0 + q : d1 + (q - K1)) * kPartialPitch + blockIdx.x] = s;
  }
  __syncthreads();
}

template <int S>
__global__ void __launch_bounds__(ORTH_NT, 1) k_arn_step(const __grid_constant__ OrthDesc d) {
  SKC_PDL_ENTRY();
  // block-uniform, before any barrier; a volatile read: the side stream's least-squares kernel
  // may raise the flag while this grid is being scheduled
  if (*reinterpret_cast<const volatile int*>(&d.st->halt)) return;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int NC = S - 1;
  extern __shared__ __align__(16) double dsm[];
  // coefficients -t [64] | reduced products [(k+1) s^2] | Gram scratch | Gram factors of the
  // k blocks | reduction scratch [16 warps][s^2 + s] | candidate slice [s-1][P]
  double* tc = dsm;
  double* hc = dsm + 64;
  double* prod = hc + kStepH;
  Gram* gs = reinterpret_cast<Gram*>(prod + orth_prod_cap(d.k, S));
  Gram* gk = gs + 1;
  double* red = reinterpret_cast<double*>(gk + d.k);
  double* sc = red + (ORTH_NT / 32) * (S * S + S);
  __shared__ int exceed[64];
  __shared__ int s_first;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * d.P;
  const int64_t rem = d.n - base;
  const int cnt = rem <= 0 ? 0 : (int)(rem < d.P ? rem : d.P);
  const int G = gridDim.x;
  auto colp = [&](int i, int l) { return d.V + ((int64_t)i * S + l) * d.np + base; };
  // this slice of candidate column j+1 (j = 0..s-2): the first kOrthSmemCols in shared memory,
  // the rest in their basis slots in global memory (C2: 124 KB of unified L1 left instead of
  // 60 KB; that capacity bounds the loads in flight per SM in every streaming phase)
  auto ccol = [&](int j) -> double* { return j < kOrthSmemCols ? sc + (int64_t)j * d.P : d.cand[j + 1] + base; };


  // Scalar2 for block i from partials (src, srcG): every CTA solves W_i t = V_i^T cand[:,1:]
  auto scalar = [&](int i, int src, int srcG, int accumulate) {
    reduce_dots_dev(d.partials, srcG, src, S * NC, prod);  // ends with __syncthreads
    if (tid < NC) {
      const int jc = tid;
      double rhs[kMaxS], t[kMaxS];
#pragma unroll
      for (int l = 0; l < S; ++l) rhs[l] = prod[l * NC + jc];
      gram_solve_t<S>(gk[i], rhs, t);
#pragma unroll
      for (int l = 0; l < S; ++l) {
        tc[l * NC + jc] = -t[l];
        if (blockIdx.x == 0) {
          double* ta = d.rec + d.rec_t + i * S * S + l * S + (jc + 1);
          *ta = accumulate ? *ta + t[l] : t[l];
        }
      }
    }
    __syncthreads();
  };

  // cand[:,1:] -= V_i t ; products V_{i+1}^T cand[:,1:] -> partials dst (when i+1 < k).
  // Points go in pairs (p, p + NT) with every basis load of the pair issued before the
  // arithmetic, so each thread keeps 2s (4s with the products) loads in flight; the products
  // still accumulate in ascending point order.
  auto round = [&](int i, int dst, bool wb, auto&& pre) {
    const bool dots = i + 1 < d.k;
    const double* Vi = colp(i, 0);
    const double* Vn = colp(dots ? i + 1 : i, 0);
    const int64_t np = d.np;
    double acc[S * NC];
#pragma unroll
    for (int q = 0; q < S * NC; ++q) acc[q] = 0.0;
    constexpr int UU = S <= 3 ? 4 : S == 4 ? SKC_UU4 : S <= 6 ? 2 : 1;
    // (with SKC_HOIST the first points' basis loads are issued before `pre` -- the reduction
    // and Gram solve of this round's coefficients -- so they are in flight during it)
    bool has[UU];
    double v[UU][S], w[UU][S];
    auto load = [&](int p0) {
#pragma unroll
      for (int u = 0; u < UU; ++u) {
        const int p = p0 + u * ORTH_NT;
        has[u] = p < cnt;
#pragma unroll
        for (int l = 0; l < S; ++l) {
          v[u][l] = has[u] ? ldcg(Vi + l * np + p) : 0.0;
          w[u][l] = dots && has[u] ? ldcg(Vn + l * np + p) : 0.0;
        }
      }
    };
#if SKC_HOIST
    load(tid);
    pre();
#else
    pre();
#endif
    for (int p0 = tid; p0 < cnt; p0 += UU * ORTH_NT) {
      double cv[UU][NC];
#if SKC_HOIST
      if (p0 != tid) load(p0);
#else
      load(p0);
#endif
#pragma unroll
      for (int u = 0; u < UU; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) cv[u][j] = has[u] ? ccol(j)[p0 + u * ORTH_NT] : 0.0;
#pragma unroll
      for (int l = 0; l < S; ++l)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const double t = tc[l * NC + j];
#pragma unroll
          for (int u = 0; u < UU; ++u) cv[u][j] = dadd(cv[u][j], dmul(t, v[u][l]));
        }
#pragma unroll
      for (int u = 0; u < UU; ++u) {
        if (!has[u]) continue;
#pragma unroll
        for (int j = 0; j < NC; ++j) ccol(j)[p0 + u * ORTH_NT] = cv[u][j];
        if (wb) {  // (the columns past kOrthSmemCols already live in their basis slots)
#pragma unroll
          for (int j = 0; j < (NC < kOrthSmemCols ? NC : kOrthSmemCols); ++j) d.cand[j + 1][base + p0 + u * ORTH_NT] = cv[u][j];
        }
        if (dots) {
#pragma unroll
          for (int l = 0; l < S; ++l)
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[l * NC + j] = fma(w[u][l], cv[u][j], acc[l * NC + j]);
        }
      }
    }
    if (dots) orth_store(acc, red, d.partials, dst);
  };

  // round-0 products V_0^T cand[:,1:] -> partials dr0 (sstep.hpp:341), four points per thread
  // with all their loads issued first
  auto r0_products = [&]() {
    constexpr int U0 = S <= 4 ? 4 : 2;
    double acc[S * NC];
#pragma unroll
    for (int q = 0; q < S * NC; ++q) acc[q] = 0.0;
    const double* V0 = colp(0, 0);
    const int64_t np = d.np;
    for (int p0 = tid; p0 < cnt; p0 += U0 * ORTH_NT) {
      double lv[U0][S], cv[U0][NC];
#pragma unroll
      for (int u = 0; u < U0; ++u) {
        const int p = p0 + u * ORTH_NT;
        const bool h = p < cnt;
#pragma unroll
        for (int l = 0; l < S; ++l) lv[u][l] = h ? ldcg(V0 + l * np + p) : 0.0;
#pragma unroll
        for (int j = 0; j < NC; ++j) cv[u][j] = h ? ccol(j)[p] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U0; ++u)
#pragma unroll
        for (int l = 0; l < S; ++l)
#pragma unroll
          for (int j = 0; j < NC; ++j) acc[l * NC + j] = fma(lv[u][l], cv[u][j], acc[l * NC + j]);
    }
    orth_store(acc, red, d.partials, d.dr0);
  };

  // L-block products with the full candidate: lhs(l) . cand[:,jc] for one block of s columns
  // (block i of the basis, or the candidate itself when i == k) -> partials d0 + l*s + jc.
  // With ZD also lhs(l) . z -> partials dz0 + l: the next block iteration's Scalar1 products
  // (z = A cand[:,s-1] of the final candidate, in memory at zg)
  auto cross_block = [&](auto zd, int i, int d0, int dz0) {
    constexpr bool ZD = decltype(zd)::value;
    // points per thread in flight, bounded by the accumulator count (no spills at 128 registers)
    constexpr int U = ZD ? (S <= 3 ? 4 : S == 4 ? 3 : S <= 6 ? 2 : 1) : (S <= 4 ? 4 : S <= 6 ? 2 : 1);
    constexpr int NA = S * S + (ZD ? S : 0);
    double acc[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) acc[q] = 0.0;
    const double* c0p = d.cand0 + base;
    const double* zg = d.z + base;
    const bool basis = i < d.k;
    const double* Li = basis ? colp(i, 0) : c0p;
    const int64_t np = d.np;
    for (int p0 = tid; p0 < cnt; p0 += U * ORTH_NT) {
      bool has[U];
      double a[U][S], b[U][S], zv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = p0 + u * ORTH_NT;
        has[u] = p < cnt;
        b[u][0] = has[u] ? ldcg(c0p + p) : 0.0;
        zv[u] = ZD && has[u] ? zg[p] : 0.0;
#pragma unroll
        for (int l = 0; l < S; ++l) a[u][l] = basis && has[u] ? ldcg(Li + l * np + p) : 0.0;
#pragma unroll
        for (int j = 1; j < S; ++j) b[u][j] = has[u] ? ccol(j - 1)[p] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!has[u]) continue;
#pragma unroll
        for (int l = 0; l < S; ++l) {
          const double av = basis ? a[u][l] : b[u][l];
#pragma unroll
          for (int jc = 0; jc < S; ++jc) acc[l * S + jc] = fma(av, b[u][jc], acc[l * S + jc]);
          if constexpr (ZD) acc[S * S + l] = fma(av, zv[u], acc[S * S + l]);
        }
      }
    }
    orth_store2<NA, S * S>(acc, red, d.partials, d0, dz0);
  };

  const int K = d.k;
  const int64_t np = d.np;
  // the previous block iteration's cross pass already produced z (in memory) and this
  // iteration's Scalar1 products (partials dz), unless it ran a reorthogonalization pass
  const bool zready = d.zfuse && K > 1 && __ldg(&d.st->zready) != 0;
  // push_block of the previous block iteration's candidate (sstep.hpp:375, 392-399) runs here,
  // off the previous kernel's tail: every CTA reduces its W (from the pass that produced the
  // candidate) and factors it in the Scalar1 phase; CTA 0 records it and stores the factor
  const bool push = K >= 2;
  if (push) reduce_dots_dev(d.partials, G, __ldg(&d.st->reorth) ? d.dwb : d.dcross + (K - 1) * S * S, S * S, tc);
  // the Gram factors of blocks 0..k-1 (k-2 with the push) into shared memory (asynchronous;
  // waited for before Scalar1)
  {
    const char* gsrc = reinterpret_cast<const char*>(d.grams);
    char* gdst = reinterpret_cast<char*>(gk);
    for (int w = tid; w < (int)((push ? K - 1 : K) * sizeof(Gram) / 8); w += ORTH_NT)
      cp_async8(gdst + 8 * w, gsrc + 8 * w, true);
    cp_async_commit();
  }
  orth_mark(d, 39);
  // ---- z = A v_{k-1}^{s-1} on this slice (the source is stable; neighbours read from memory)
  // y = A x on this slice; xs (optional) is this slice of x in shared memory, read in place of
  // memory for the points it covers.  The 2D constant stencil takes a 32-bit fast path (same
  // arithmetic: S, W, C, E, N in ascending column order, absent neighbours skipped).
  // xscale (when nonzero) multiplies every source value as it is read (the source is then
  // seed and the values level 0 = seed / nu, rounded exactly as when stored); put(p, y, x_p)
  // also receives the point's own source value
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
  // z and seed of this slice stay in shared memory (candidate columns 0 and s-2, free until
  // the powers reach them; with s = 2 seed also goes to memory for its neighbours)
  double* zs = sc;
  double* seeds = nullptr;  // (the column that used to hold it is now in global memory)
  if (zready) {
    for (int p = tid; p < cnt; p += ORTH_NT) zs[p] = d.z[base + p];
  } else {
    apply_slice(d.vin, nullptr, 0.0, [&](int p, double v, double) { zs[p] = v; });
  }
  orth_mark(d, 40);
  // ---- Scalar1 products V_i^T z (i < k) -> dz + i s + l, and z.z -> dz + k s (each thread
  //      reads back its own z); blocks in descending order, so the seed sweep's first blocks
  //      are still in L2
  if (!zready) {
    double zz[1] = {0.0};
    for (int i = K - 1; i >= 0; --i) {
      double acc[S];
#pragma unroll
      for (int q = 0; q < S; ++q) acc[q] = 0.0;
      const double* Vi = colp(i, 0);
      for (int p0 = tid; p0 < cnt; p0 += ORTH_UC * ORTH_NT) {
        double zv[ORTH_UC], v[ORTH_UC][S];
#pragma unroll
        for (int u = 0; u < ORTH_UC; ++u) {
          const int p = p0 + u * ORTH_NT;
          const bool h = p < cnt;
          zv[u] = h ? zs[p] : 0.0;
#pragma unroll
          for (int l = 0; l < S; ++l) v[u][l] = h ? ldcg(Vi + l * np + p) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < ORTH_UC; ++u) {
          if (p0 + u * ORTH_NT >= cnt) continue;
#pragma unroll
          for (int l = 0; l < S; ++l) acc[l] = fma(v[u][l], zv[u], acc[l]);
          if (i == 0) zz[0] = fma(zv[u], zv[u], zz[0]);
        }
      }
      orth_store(acc, red, d.partials, d.dz + i * S);
    }
    orth_store(zz, red, d.partials, d.dz + K * S);
  }
  orth_mark(d, 6);
  orth_mark_all(d, 256);
  if (!zready) grid.sync();  // (with zready the products come from the previous launch)
  // ---- Scalar1 (sstep.hpp:301-310): zn, h_i = W_i^{-1} V_i^T z in every CTA (Gram factors
  // from shared memory); CTA 0 records
  cp_async_wait<0>();
  reduce_dots_dev(d.partials, G, d.dz, K * S + 1, prod);  // (ends with __syncthreads)
  if (push) {
    __shared__ int s_push_ok;
    if (tid == 0) {
      const bool ok = arn_push_body<S>(d.st, gk[K - 1], K - 1, d.rec_push, tc, S, blockIdx.x == 0);
      s_push_ok = ok;
      if (ok && blockIdx.x == 0) d.grams[K - 1] = gk[K - 1];
    }
    __syncthreads();
    if (!s_push_ok) return;  // basis collapse (identical decision in every CTA)
  }
  const double zn = sqrt(prod[K * S]);
  if (blockIdx.x == 0 && tid == 0) {
    d.rec[RecLayout::kZn] = zn;
    d.rec[RecLayout::kReorth] = 0.0;
    d.rec[RecLayout::kFirst] = -1.0;
  }
  for (int i = tid; i < K; i += ORTH_NT) {
    double rhs[kMaxS], h[kMaxS];
    for (int l = 0; l < S; ++l) rhs[l] = prod[i * S + l];
    gram_solve_t<S>(gk[i], rhs, h);
    for (int l = 0; l < S; ++l) {
      hc[i * S + l] = -h[l];
      if (blockIdx.x == 0) d.rec[d.rec_h + i * S + l] = h[l];
    }
  }
  __syncthreads();
  orth_mark(d, 41);
  // ---- seed = z - sum_i V_i h_i (terms in block order, multiply and add rounded separately),
  //      one sweep per block with the running sum in shared memory (every point stays with
  //      its thread), then ||seed||^2
  {
    for (int i = 0; i < K; ++i) {
      const double* Vi = colp(i, 0);
      double hl[S];
#pragma unroll
      for (int l = 0; l < S; ++l) hl[l] = hc[i * S + l];
      for (int p0 = tid; p0 < cnt; p0 += ORTH_UC * ORTH_NT) {
        double v[ORTH_UC][S], o[ORTH_UC];
#pragma unroll
        for (int u = 0; u < ORTH_UC; ++u) {
          const int p = p0 + u * ORTH_NT;
          const bool h = p < cnt;
          o[u] = h ? zs[p] : 0.0;
#pragma unroll
          for (int l = 0; l < S; ++l) v[u][l] = h ? ldcg(Vi + l * np + p) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < ORTH_UC; ++u) {
          const int p = p0 + u * ORTH_NT;
          if (p >= cnt) continue;
#pragma unroll
          for (int l = 0; l < S; ++l) o[u] = dadd(o[u], dmul(hl[l], v[u][l]));
          zs[p] = o[u];
        }
      }
    }
    double acc[1] = {0.0};
    for (int p = tid; p < cnt; p += ORTH_NT) {
      const double o = zs[p];
      d.seed[base + p] = o;
      if (seeds) seeds[p] = o;
      acc[0] = fma(o, o, acc[0]);
    }
    orth_store(acc, red, d.partials, d.dseed);
  }
  orth_mark(d, 7);
  orth_mark_all(d, 512);
  grid.sync();
  // ---- nu = ||seed|| and the invariant-subspace test (sstep.hpp:315-324)
  reduce_dots_dev(d.partials, G, d.dseed, 1, prod);
  const double nu = sqrt(prod[0]);
  if (blockIdx.x == 0 && tid == 0) d.rec[RecLayout::kNu] = nu;
  if (nu <= 1e-14 * zn) {  // identical decision in every CTA
    if (blockIdx.x == 0 && tid == 0) {
      d.rec[RecLayout::kInv] = 1.0;
      d.st->status = kArnInvariant;
      d.st->block = K;
      d.st->halt = 1;
    }
    return;
  }
  const double inv = 1.0 / nu;
  orth_mark(d, 42);
  // ---- candidate block [v, A v, .., A^{s-1} v], v = seed / nu (krylov_block, block.hpp:59-67):
  //      every level is an exact spmv of the previous one; levels 1..s-1 stay in shared memory,
  //      levels 0..s-2 also go to memory for the neighbours' next level
  orth_mark(d, 44);
  if (S <= 4 && d.spow) {
    // Row-streamed: the slice is walked in index rows of nx points (row r = [r nx, (r+1) nx)
    // relative to the slice start); step k computes level j on row k - 2(j-1), so every level
    // only reads rows of the previous level finished in earlier steps (one __syncthreads per
    // step, no grid barrier).  Level j is computed on e_j = s-1-j ghost rows beyond each slice
    // edge, redundantly with the neighbouring CTAs (level 1 from seed / nu in memory), so the
    // slice's last level needs nothing from other CTAs.  Ghost rows live in small per-CTA global buffers
    // (the bottom ghosts are dead before the top ghosts are written, so both share one buffer;
    // the host enables this only when every slice has at least 4 rows).  Each point is the
    // same ascending-column sum as spmv, so the levels are bit-identical to the sweeps.
    const int nx = (int)d.op.nx, ny = (int)d.op.ny;
    const double cS = d.op.coef[1], cW = d.op.coef[2], cC = d.op.coef[3], cE = d.op.coef[4], cN = d.op.coef[5];
    double* gh[2] = {d.ghosts + (int64_t)blockIdx.x * (d.g1 + d.g2), d.ghosts + (int64_t)blockIdx.x * (d.g1 + d.g2) + d.g1};
    const int Rs = cnt > 0 ? (cnt + nx - 1) / nx : 0;
    int ic[2], jc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t q = base + 2 * tid + h;
      ic[h] = (int)(q % nx);
      jc[h] = (int)(q / nx);
    }
    // level j value at relative index v (slice, or the level's ghost buffer)
    auto slot = [&](int j, int v) -> double* {
      if (v >= 0 && v < cnt) return ccol(j - 1) + v;
      const int e = S - 1 - j;
      return gh[j - 1] + (v < 0 ? v + e * nx : v - cnt);
    };
    const int kend = cnt > 0 ? Rs - 1 + 2 * (S - 2) : -(S - 2) - 1;
    const int rin = cnt == Rs * nx ? Rs - 2 : Rs - 3;  // last row whose north neighbours are in the slice
    // level 1's source rows (seed, columns c0-1 .. c0+2 of this thread's pair) in a register
    // ring: rows k-1, k, k+1 in use, row k+2 loaded one step ahead
    const int c0 = 2 * tid;
    const int64_t q00 = base + c0;  // global index of (row 0, column c0)
    auto load_row = [&](int rr, double (&o)[4]) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int64_t q = q00 + (int64_t)rr * nx + t - 1;
        o[t] = c0 < nx && q >= 0 && q < d.n ? __ldcg(d.seed + q) : 0.0;
      }
    };
    double ra[4], rb[4], rc[4], rn[4];
    load_row(-(S - 2) - 1, ra);
    load_row(-(S - 2), rb);
    load_row(-(S - 2) + 1, rc);
    for (int k = -(S - 2); k <= kend; ++k) {
      load_row(k + 2, rn);  // (in flight during this step)
#pragma unroll
      for (int j = S - 1; j >= 1; --j) {
        const int r = k - 2 * (j - 1), e = S - 1 - j;
        if (r < -e || r > Rs - 1 + e) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = c0 + h;
          if (c >= nx) continue;
          const int v = r * nx + c;
          const int jr = jc[h] + r, i = ic[h];
          if (v < -e * nx || v >= cnt + e * nx || jr < 0 || jr >= ny) continue;
          double xs_, xw_, xc_, xe_, xn_;
          if (j == 1) {  // seed / nu from the ring (multiply rounded as when level 0 is stored)
            xs_ = __dmul_rn(ra[h + 1], inv);
            xw_ = __dmul_rn(rb[h], inv);
            xc_ = __dmul_rn(rb[h + 1], inv);
            xe_ = __dmul_rn(rb[h + 2], inv);
            xn_ = __dmul_rn(rc[h + 1], inv);
          } else if (r >= 1 && r <= rin) {  // every neighbour inside the slice: shared memory
            const double* Pj = ccol(j - 2) + v;
            xs_ = Pj[-nx];
            xw_ = Pj[-1];
            xc_ = Pj[0];
            xe_ = Pj[1];
            xn_ = Pj[nx];
          } else {
            xs_ = jr > 0 ? *slot(j - 1, v - nx) : 0.0;
            xw_ = i > 0 ? *slot(j - 1, v - 1) : 0.0;
            xc_ = *slot(j - 1, v);
            xe_ = i + 1 < nx ? *slot(j - 1, v + 1) : 0.0;
            xn_ = jr + 1 < ny ? *slot(j - 1, v + nx) : 0.0;
          }
          double a = 0.0;
          if (jr > 0) a = __dadd_rn(a, __dmul_rn(cS, xs_));
          if (i > 0) a = __dadd_rn(a, __dmul_rn(cW, xw_));
          a = __dadd_rn(a, __dmul_rn(cC, xc_));
          if (i + 1 < nx) a = __dadd_rn(a, __dmul_rn(cE, xe_));
          if (jr + 1 < ny) a = __dadd_rn(a, __dmul_rn(cN, xn_));
          if (r >= 1 && r <= rin)
            ccol(j - 1)[v] = a;
          else
            *slot(j, v) = a;
          if (v >= 0 && v < cnt) {
            if (j == 1) d.cand[0][base + v] = xc_;
            if (!d.build_next) d.cand[j][base + v] = a;
          }
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) ra[t] = rb[t], rb[t] = rc[t], rc[t] = rn[t];
      __syncthreads();
    }
  } else
  // level 1 reads seed / nu on the fly (level 0 is stored by the same sweep); levels >= 2 read
  // their source from shared memory inside the slice
  for (int j = 1; j < S; ++j) {
    if (j > 1) grid.sync();
    orth_mark(d, 44 + 2 * j - 1);
    const bool to_mem = j + 1 < S || !d.build_next;
    apply_slice(j == 1 ? d.seed : d.cand[j - 1], j >= 2 && j - 2 < kOrthSmemCols ? ccol(j - 2) : seeds, j == 1 ? inv : 0.0,
                [&](int p, double v, double xc) {
                  if (j == 1) d.cand[0][base + p] = xc;
                  ccol(j - 1)[p] = v;
                  if (to_mem) d.cand[j][base + p] = v;
                });
    orth_mark(d, 44 + 2 * j);
  }
  orth_mark(d, 43);
  if (!d.build_next) return;  // the last block iteration builds the candidate only
  // ---- round-0 products V_0^T cand[:,1:] (sstep.hpp:341)
  r0_products();
  grid.sync();
  orth_mark(d, 0);
  // ---- pass 0; the last round also writes the candidate back (final unless a second pass
  //      runs) and, with zfuse, is followed by a barrier so z = A cand[:,s-1] can be formed
  for (int i = 0; i < K; ++i) {
    round(i, ((i + 1) & 1) ? d.dr1 : d.dr0, i + 1 == K, [&] {
      scalar(i, (i & 1) ? d.dr1 : d.dr0, G, 0);
      orth_mark(d, 8 + 3 * i);
    });
    orth_mark(d, 9 + 3 * i);
    if (i + 1 < K || d.zfuse) grid.sync();
    orth_mark(d, 10 + 3 * i);
  }
  // ---- the next block iteration's z = A cand[:,s-1] (to memory) and z.z -> dz + (k+1) s
  if (d.zfuse) {
    double zz[1] = {0.0};
    double* zg = d.z + base;
    apply_slice(d.cand[S - 1], nullptr, 0.0, [&](int p, double v, double) {
      zg[p] = v;
      zz[0] = fma(v, v, zz[0]);
    });
    orth_store(zz, red, d.partials, d.dz + (K + 1) * S);
  }
  orth_mark(d, 60);
  // ---- cross products and W (needs_reorth, sstep.hpp:401-414), with zfuse also the next
  //      iteration's Scalar1 products [V_0..V_{k-1}, cand]^T z; blocks in descending order (the
  //      last rounds' blocks are still in L2, and the next seed sweep starts at block 0)
  for (int i = K; i >= 0; --i) {
    if (d.zfuse)
      cross_block(std::true_type{}, i, d.dcross + i * S * S, d.dz + i * S);
    else
      cross_block(std::false_type{}, i, d.dcross + i * S * S, 0);
  }
  orth_mark(d, 1);
  orth_mark_all(d, 768);
  grid.sync();
  orth_mark(d, 2);
  reduce_dots_dev(d.partials, G, d.dcross, (K + 1) * S * S, prod);
  {
    const double* sW = prod + K * S * S;
    double cn2 = 0.0;
    for (int jc = 0; jc < S; ++jc) cn2 += sW[jc * S + jc];
    for (int i = tid; i < K; i += ORTH_NT) {
      const double* cr = prod + i * S * S;
      double acc = 0.0;
      for (int q = 0; q < S * S; ++q) acc += cr[q] * cr[q];
      exceed[i] = sqrt(acc) > d.orth_tol * sqrt(sd_trace(gk[i].w, S)) * sqrt(cn2);
    }
    __syncthreads();
    if (tid == 0) {
      int first = -1;
      for (int i = 0; i < K; ++i)
        if (exceed[i]) {
          first = i;
          break;
        }
      s_first = first;
      if (blockIdx.x == 0) {
        d.rec[RecLayout::kFirst] = first;
        d.rec[RecLayout::kReorth] = first >= 0 ? 1.0 : 0.0;
        d.st->reorth = first >= 0;
        d.st->zready = d.zfuse && first < 0;
      }
    }
    __syncthreads();
  }
  orth_mark(d, 3);
  if (s_first >= 0) {
    // ---- pass 1: V_0^T cand[:,1:], k rounds with t accumulated, then W of the new candidate
    r0_products();
    grid.sync();
    for (int i = 0; i < K; ++i) {
      round(i, ((i + 1) & 1) ? d.dr1 : d.dr0, i + 1 == K, [&] { scalar(i, (i & 1) ? d.dr1 : d.dr0, G, 1); });
      if (i + 1 < K) grid.sync();
    }
    cross_block(std::false_type{}, K, d.dwb, 0);
    grid.sync();
    orth_mark(d, 4);
    // the candidate's raw Gram products for the least-squares stream (its snapshot: the next
    // block iteration reuses the partial regions)
    if (blockIdx.x == 0) {
      reduce_dots_dev(d.partials, G, d.dwb, S * S, tc);  // (ends with a barrier)
      if (tid < S * S) d.rec[d.rec_wraw + tid] = tc[tid];
    }
  } else {
    orth_mark(d, 4);
    if (blockIdx.x == 0 && tid < S * S) d.rec[d.rec_wraw + tid] = prod[K * S * S + tid];
  }
  orth_mark(d, 5);
}

size_t orth_smem(int s, int k, int64_t P) {
  return sizeof(double) * (64 + kStepH + (size_t)orth_prod_cap(k, s)) + sizeof(Gram) * (1 + (size_t)k) +
         sizeof(double) * (ORTH_NT / 32) * (s * s + s) +
         sizeof(double) * (size_t)std::min(s - 1, kOrthSmemCols) * (size_t)P;
}

// ghost-row buffer sizes (doubles) of the row-streamed powers for slices of P points, or
// false when they do not apply (the 2D constant stencil, s <= 4, nx <= 2 x threads, every
// non-empty slice at least 4 rows)
bool stream_powers_ghosts(const DevOp& op, int s, int64_t n, int64_t P, int G, int& g1, int& g2) {
  g1 = g2 = 0;
  if (op.kind != kStencilConst || op.dim != 2 || s < 2 || s > 4 || op.nx > 2 * ORTH_NT) return false;
  const int64_t nx = op.nx;
  for (int b = 0; b < G; ++b) {
    const int64_t base = (int64_t)b * P;
    if (base >= n) break;
    const int64_t cnt = std::min(P, n - base);
    const int64_t Rs = (cnt + nx - 1) / nx;
    if (Rs < 4) return false;
    for (int j = 1; j <= s - 2; ++j) {
      const int64_t e = s - 1 - j;
      const int64_t need = std::max(e * nx, (Rs + e) * nx - cnt);
      int& g = j == 1 ? g1 : g2;
      g = (int)std::max<int64_t>(g, need);
    }
  }
  return true;
}

template <int S>
void run_orth(Ctx& c, const OrthDesc& d, int G, size_t smem) {
  // (at most 227 KB per block less the kernel's static shared memory; orth_points caps smem)
  ensure_smem(k_arn_step<S>, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = G;
  cfg.blockDim = ORTH_NT;
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
  int64_t orth_points() const {
    if (!c.orth || c.world() != 1 || g.grouped() || s < 2 || op.d.kind == kIlu0) return 0;
    const int64_t P = ((op.n + mk_ctas() - 1) / mk_ctas() + 1) & ~(int64_t)1;
    return orth_smem(s, m, P) <= kOrthSmemCap ? P : 0;
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
    // (off by default: the fused products make the cross pass and the extra barrier cost
    // about what the skipped Scalar1 sweep saves, measured 0.5-0.8% slower on C2)
    d.zfuse = build_next && c.zfuse ? 1 : 0;
    d.n = op.n;
    d.P = orth_points();
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
    static const bool trace = std::getenv("SKC_TRACE_ORTH") != nullptr;
    if (trace) d.trace = (unsigned long long*)c.workspace("orth_trace", 1024 * sizeof(unsigned long long));
    const int G = mk_ctas();
    int g1 = 0, g2 = 0;
    d.spow = c.spow && stream_powers_ghosts(op.d, s, op.n, d.P, G, g1, g2);
    d.g1 = d.spow ? g1 : 0;
    d.g2 = d.spow ? g2 : 0;
    if (d.spow) d.ghosts = (double*)c.workspace("orth_ghosts", sizeof(double) * (size_t)G * (g1 + g2));
    const size_t smem = orth_smem(s, k, d.P);
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
        if (!have) {
          std::vector<const double*> L;
          for (int l = 0; l < s; ++l) L.push_back(col(0, l));
          launch_gram_list(c, g, L, Cr, partials, dl.D(), halt, cond, pass ? "gram_mgs_reorth" : "gram_mgs");
        }
        for (int i = 0; i < k; ++i) {
          const int Gi = (i == 0 && have) ? Gfused : g.enc();
          // Scalar2 against block i (sstep.hpp:338-353) runs in the update kernel's prologue:
          // t = W_i^{-1} V_i^T cand[:,1:], recorded at block i of this iteration's T area
          const MgsScalar sc{partials, c.reduce_point(partials, Gi, dl.Dr(i), s * (s - 1)), dl.Dr(i), grams + i,
                             tk + i * s * s, pass};
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
          launch_k(c, k_arn_check, 1, 256, 0, st, grams, k, rk, partials, c.reduce_point(partials, g.enc(), dl.Cross(), k * s * s + s * s), dl.Cross(), dl.Cross() + k * s * s, s, 1e-8, scratch);
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
