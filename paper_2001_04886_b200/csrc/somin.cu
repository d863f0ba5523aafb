// somin.cu -- device-resident s-step Orthomin(k) / s-GCR (sstep.hpp:142-249) and s-MR
// (sstep.hpp:89-135).
//
// All n-length work runs on the GPU; the s x s Gram factorizations/solves and every
// termination decision run in single-CTA "scalar" kernels on the device (same IEEE
// arithmetic as the host reference, small_dense.cuh), so the host enqueues whole batches
// of iterations and synchronizes once per batch.  A device halt flag turns every later
// kernel of the batch into a no-op once the iteration stops.  The host then replays the
// reference's control flow on the recorded per-iteration residuals to rebuild the
// SolveReport (history, op counters, breakdown strings) exactly.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "device_util.cuh"
#include "solver_util.hpp"
#include "stencil.cuh"

namespace skc {

namespace {

enum : int {
  kRunning = 0,
  kConverged = 1,
  kDiverged = 2,
  kMaxIter = 3,
  kSetupCollapse = 4,
  kIterCollapse = 5,
  kLogic = 6,
  kNanStop = 7,
};

struct SominState {
  int status;
  int halt;
  int singular1;
  int fixed;  // fixed-step benchmark mode (gram_bypass_ratio)
  long long iters;
  long long max_iter;
  double tol, divf, r0n, rn, ratio;
};

constexpr int kMaxWin = 128;  // window entries addressable by one scalar kernel
struct Slots {
  int n;
  int16_t idx[kMaxWin];
};

// coefficient layout
__host__ __device__ constexpr int cA(int) { return 0; }
__host__ __device__ constexpr int cNegA(int s) { return s; }
__host__ __device__ constexpr int cMinus1(int s) { return 2 * s; }
__host__ __device__ constexpr int cB(int s) { return 2 * s + 1; }

__global__ void k_somin_start(SominState* st, const double* partials, int G, int d0) {
  SKC_PDL_ENTRY();
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    const double rn = sqrt(v[0]);
    st->r0n = rn;
    st->rn = rn;
    if (!(rn > st->tol)) {
      st->status = rn <= st->tol ? kConverged : kNanStop;
      st->halt = 1;
    }
  }
}

// Factor W (full s x s from dot region dW, symmetrized like block_gram_self) into grams[slot]
// and solve a = W^{-1} m.  Shared by setup and push.
__device__ void somin_factor_solve(SominState* st, Gram* gslot, double* coef, const double* W, const double* m,
                                   int s, int collapse_status) {
  Gram g;
  gram_factor_dev(g, W, s);
  gram_bypass_ratio(g, st->fixed);
  if (!g.ok) {
    st->status = collapse_status;
    st->halt = 1;
    st->ratio = g.ratio;
    st->singular1 = g.singular1;
    return;
  }
  *gslot = g;
  double a[kMaxS];
  gram_solve_dev(g, m, a);
  for (int l = 0; l < s; ++l) {
    coef[cA(s) + l] = a[l];
    coef[cNegA(s) + l] = -a[l];
  }
}

// setup: W0 = gram(AR0, AR0) (s*s dots, full), m0 = AR0^T r (s dots)
__global__ void k_somin_setup(SominState* st, Gram* grams, double* coef, const double* partials, int G, int dW,
                              int dm, int s) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[kMaxS * kMaxS + kMaxS];
  reduce_dots_dev(partials, G, dW, s * s, v);
  reduce_dots_dev(partials, G, dm, s, v + s * s);
  if (threadIdx.x == 0) {
    double W[kMaxS * kMaxS];
    for (int j = 0; j < s; ++j)
      for (int l = 0; l < s; ++l) W[j * s + l] = v[j * s + l];
    for (int j = 0; j < s; ++j)
      for (int l = j + 1; l < s; ++l) {  // block.hpp:80-91 averaging (exact: dots are symmetric)
        const double avg = (W[j * s + l] + W[l * s + j]) / 2.0;
        W[j * s + l] = avg;
        W[l * s + j] = avg;
      }
    coef[cMinus1(s)] = -1.0;
    somin_factor_solve(st, &grams[0], coef, W, v + s * s, s, kSetupCollapse);
  }
}

__global__ void k_somin_norm(SominState* st, const double* partials, int G, int d0, double* hist) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    const double rn = sqrt(v[0]);
    st->rn = rn;
    st->iters += 1;
    hist[st->iters] = rn;
    int status = kRunning;
    if (rn <= st->tol)
      status = kConverged;
    else if (rn > st->divf * st->r0n)
      status = kDiverged;
    else if (st->iters >= st->max_iter)
      status = kMaxIter;
    if (status) {
      st->status = status;
      st->halt = 1;
    }
  }
}

// Scalar2 (sstep.hpp:204-214): b_e = -W_e^{-1} C_e for every window entry e
__global__ void k_somin_proj(SominState* st, const Gram* grams, const __grid_constant__ Slots win, double* coef,
                             const double* partials, int G, int dC, int s, double* scratch) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  reduce_dots_dev(partials, G, dC, win.n * s * s, scratch);
  for (int t = threadIdx.x; t < win.n * s; t += blockDim.x) {
    const int e = t / s, jc = t % s;
    double rhs[kMaxS], x[kMaxS];
    for (int l = 0; l < s; ++l) rhs[l] = scratch[(e * s + l) * s + jc];
    gram_solve_dev(grams[win.idx[e]], rhs, x);
    for (int l = 0; l < s; ++l) coef[cB(s) + e * s * s + l * s + jc] = -x[l];
  }
}

// W (upper triangle, tri order) + m of the new block; optional debug A-orthogonality check
// (sstep.hpp:225-233), then GramSolver (breakdown = basis collapse) and a = W^{-1} m.
__global__ void k_somin_push(SominState* st, Gram* grams, int slot_new, double* coef, const double* partials, int G,
                             int dW, int dm, int s, int debug, const __grid_constant__ Slots win, int dX,
                             double* scratch) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  const int ntri = s * (s + 1) / 2;
  reduce_dots_dev(partials, G, dW, ntri, scratch);
  reduce_dots_dev(partials, G, dm, s, scratch + ntri);
  if (debug) reduce_dots_dev(partials, G, dX, win.n * s * s, scratch + ntri + s);
  if (threadIdx.x == 0) {
    double W[kMaxS * kMaxS];
    int t = 0;
    for (int a = 0; a < s; ++a)
      for (int b = a; b < s; ++b) {
        W[a * s + b] = scratch[t];
        W[b * s + a] = scratch[t];
        ++t;
      }
    if (debug) {
      const double nn = sqrt(sd_trace(W, s));
      for (int e = 0; e < win.n; ++e) {
        const double* cr = scratch + ntri + s + e * s * s;
        double acc = 0.0;
        for (int q = 0; q < s * s; ++q) acc += cr[q] * cr[q];
        if (sqrt(acc) > 1e-7 * nn * sqrt(sd_trace(grams[win.idx[e]].w, s))) {
          st->status = kLogic;
          st->halt = 1;
          return;
        }
      }
    }
    somin_factor_solve(st, &grams[slot_new], coef, W, scratch + ntri, s, kIterCollapse);
    if (!st->halt && !(st->rn > st->tol)) {  // NaN residual: the loop condition ends the solve
      st->status = kNanStop;
      st->halt = 1;
    }
  }
}

// ---------------------------------------------------------------- persistent s-Omin (small n)
// For problems whose vectors are L2-resident and too small to fill the GPU with one kernel per
// operation (C1: 16 384 unknowns), one cooperative launch runs a chunk of whole s-Omin
// iterations: every CTA owns a contiguous point range and the phases of an iteration are
// separated by grid barriers instead of kernel boundaries --
//   x += P a, r -= AP a and ||r||^2 | norm, termination checks | the s powers of r (a barrier
//   between levels) and C_e = AP_e^T AR | Scalar2 solves in every CTA | the new P, AP block,
//   W and m | push_block (factor in every CTA; CTA 0 records) and a = W^{-1} m.
// Every CTA reduces the per-CTA partials in the same fixed order and takes the same decisions;
// CTA 0 writes the state and the history.  The window slots follow the host deque exactly:
// the block of iteration t lives in slot t mod (k+1), the window before iteration t's push is
// the blocks of iterations max(0, t-k) .. t-1.  Same per-element arithmetic as the batched path.
constexpr int PS_NT = 256;
constexpr int PS_MAXK = 8;

struct PersistDesc {
  DevOp op;
  int k;
  int64_t n, P, np;
  double* x;
  double* r;
  double* K;   // powers: column j at K + j*np
  double* S0;  // slot 0 column 0; slot sl column col (P: col < s, AP: s + col) at S0 + (sl*2s + col)*np
  double* partials;
  int dRR, dW, dC;
  Gram* grams;
  double* coef;
  SominState* st;
  double* hist;
  long long it_end;
};

template <int K>
__device__ __forceinline__ void ps_store(const double (&acc)[K], double* red, double* partials, int d0) {
  constexpr int NW = PS_NT / 32;
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

template <int S>
__global__ void __launch_bounds__(PS_NT) k_somin_persist(const __grid_constant__ PersistDesc d) {
  SKC_PDL_ENTRY();
  if (__ldg(&d.st->halt)) return;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int NTRI = S * (S + 1) / 2;
  __shared__ Gram gw[PS_MAXK + 1];
  __shared__ double sa[S], sb[PS_MAXK * S * S], sv[PS_MAXK * S * S + NTRI + S];
  __shared__ double red[(PS_NT / 32) * (NTRI + S > S * S ? NTRI + S : S * S)];
  __shared__ int s_flag;
  const int tid = threadIdx.x, G = gridDim.x, NSL = d.k + 1;
  const int64_t base = (int64_t)blockIdx.x * d.P;
  const int cnt = base >= d.n ? 0 : (int)(d.n - base < d.P ? d.n - base : d.P);
  for (int w = tid; w < (int)(NSL * sizeof(Gram) / 8); w += PS_NT)
    reinterpret_cast<uint64_t*>(gw)[w] = reinterpret_cast<const uint64_t*>(d.grams)[w];
  if (tid < S) sa[tid] = d.coef[cA(S) + tid];
  const double tol = d.st->tol, divf = d.st->divf, r0n = d.st->r0n;
  const long long max_iter = d.st->max_iter;
  long long t = d.st->iters;
  __syncthreads();
  auto pcol = [&](int sl, int col) { return d.S0 + ((int64_t)sl * 2 * S + col) * d.np; };
  auto kcol = [&](int j) { return d.K + (int64_t)j * d.np; };
  for (;;) {
    // ---- x += P a ; r -= AP a ; ||r||^2 (sstep.hpp:183-193)
    {
      const int cur = (int)(t % NSL);
      double rr[1] = {0.0};
      for (int p = tid; p < cnt; p += PS_NT) {
        const int64_t q = base + p;
        double xv = d.x[q], rv = d.r[q];
#pragma unroll
        for (int l = 0; l < S; ++l) xv = __dadd_rn(xv, __dmul_rn(sa[l], pcol(cur, l)[q]));
#pragma unroll
        for (int l = 0; l < S; ++l) rv = __dadd_rn(rv, __dmul_rn(-sa[l], pcol(cur, S + l)[q]));
        d.x[q] = xv;
        d.r[q] = rv;
        rr[0] = fma(rv, rv, rr[0]);
      }
      ps_store(rr, red, d.partials, d.dRR);
    }
    grid.sync();
    reduce_dots_dev(d.partials, G, d.dRR, 1, sv);
    ++t;
    const double rn = sqrt(sv[0]);
    {
      int status = kRunning;
      if (rn <= tol)
        status = kConverged;
      else if (rn > divf * r0n)
        status = kDiverged;
      else if (t >= max_iter)
        status = kMaxIter;
      if (blockIdx.x == 0 && tid == 0) {
        d.st->rn = rn;
        d.st->iters = t;
        d.hist[t] = rn;
        if (status) {
          d.st->status = status;
          d.st->halt = 1;
        }
      }
      if (status) return;
    }
    // ---- krylov_pair(r): K[j] = A^{j+1} r (every level an exact spmv of the previous one)
#pragma unroll 1
    for (int j = 0; j < S; ++j) {
      const double* src = j == 0 ? d.r : kcol(j - 1);
      double* dst = kcol(j);
      for (int p = tid; p < cnt; p += PS_NT) {
        const int64_t q = base + p;
        GridWalk w;
        w.init(d.op, q);
        dst[q] = apply_point(d.op, [&](int64_t o) { return src[o]; }, q, w);
      }
      if (j + 1 < S) grid.sync();
    }
    // ---- C_e = AP_e^T AR for the window (block_gram, sstep.hpp:207); own points only
    const int nw = (int)(t < d.k ? t : d.k);  // window blocks: iterations t - nw .. t - 1
#pragma unroll 1
    for (int e = 0; e < nw; ++e) {
      const int se = (int)((t - nw + e) % NSL);
      double acc[S * S];
#pragma unroll
      for (int q2 = 0; q2 < S * S; ++q2) acc[q2] = 0.0;
      for (int p = tid; p < cnt; p += PS_NT) {
        const int64_t q = base + p;
        double kv[S];
#pragma unroll
        for (int jc = 0; jc < S; ++jc) kv[jc] = kcol(jc)[q];
#pragma unroll
        for (int l = 0; l < S; ++l) {
          const double ap = pcol(se, S + l)[q];
#pragma unroll
          for (int jc = 0; jc < S; ++jc) acc[l * S + jc] = fma(ap, kv[jc], acc[l * S + jc]);
        }
      }
      ps_store(acc, red, d.partials, d.dC + e * S * S);
    }
    grid.sync();
    // ---- Scalar2 (sstep.hpp:204-214): b_e = -W_e^{-1} C_e in every CTA
    reduce_dots_dev(d.partials, G, d.dC, nw * S * S, sv);
    for (int u = tid; u < nw * S; u += PS_NT) {
      const int e = u / S, jc = u % S;
      const int se = (int)((t - nw + e) % NSL);
      double rhs[kMaxS], xx[kMaxS];
#pragma unroll
      for (int l = 0; l < S; ++l) rhs[l] = sv[(e * S + l) * S + jc];
      gram_solve_t<S>(gw[se], rhs, xx);
#pragma unroll
      for (int l = 0; l < S; ++l) sb[e * S * S + l * S + jc] = -xx[l];
    }
    __syncthreads();
    // ---- new block P = R + sum_e P_e b_e, AP = AR + sum_e AP_e b_e (window block -> column l
    //      order, sstep.hpp:215-221), W = AP^T AP (upper triangle) and m = AP^T r
    const int nsl = (int)(t % NSL);
    {
      double acc[NTRI + S];
#pragma unroll
      for (int q2 = 0; q2 < NTRI + S; ++q2) acc[q2] = 0.0;
      for (int p = tid; p < cnt; p += PS_NT) {
        const int64_t q = base + p;
        const double rv = d.r[q];
        double pn[S], apn[S];
#pragma unroll
        for (int jc = 0; jc < S; ++jc) {
          pn[jc] = jc == 0 ? rv : kcol(jc - 1)[q];
          apn[jc] = kcol(jc)[q];
        }
        for (int e = 0; e < nw; ++e) {
          const int se = (int)((t - nw + e) % NSL);
          const double* be = sb + e * S * S;
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double pv = pcol(se, l)[q];
#pragma unroll
            for (int jc = 0; jc < S; ++jc) pn[jc] = __dadd_rn(pn[jc], __dmul_rn(be[l * S + jc], pv));
          }
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const double apv = pcol(se, S + l)[q];
#pragma unroll
            for (int jc = 0; jc < S; ++jc) apn[jc] = __dadd_rn(apn[jc], __dmul_rn(be[l * S + jc], apv));
          }
        }
#pragma unroll
        for (int jc = 0; jc < S; ++jc) {
          pcol(nsl, jc)[q] = pn[jc];
          pcol(nsl, S + jc)[q] = apn[jc];
        }
        int u = 0;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int b = a; b < S; ++b) acc[u] = fma(apn[a], apn[b], acc[u]), ++u;
#pragma unroll
        for (int a = 0; a < S; ++a) acc[NTRI + a] = fma(apn[a], rv, acc[NTRI + a]);
      }
      ps_store(acc, red, d.partials, d.dW);
    }
    grid.sync();
    // ---- push_block: GramSolver(W) (breakdown = basis collapse) and a = W^{-1} m
    reduce_dots_dev(d.partials, G, d.dW, NTRI + S, sv);
    if (tid == 0) {
      double W[S * S];
      int u = 0;
#pragma unroll
      for (int a = 0; a < S; ++a)
#pragma unroll
        for (int b = a; b < S; ++b) {
          W[a * S + b] = sv[u];
          W[b * S + a] = sv[u];
          ++u;
        }
      gram_factor_t<S>(gw[nsl], W);
      gram_bypass_ratio(gw[nsl], d.st->fixed);
      int flag = 0;
      if (!gw[nsl].ok) {
        flag = kIterCollapse;
      } else {
        double a[kMaxS];
        gram_solve_t<S>(gw[nsl], sv + NTRI, a);
#pragma unroll
        for (int l = 0; l < S; ++l) sa[l] = a[l];
        if (!(rn > tol)) flag = kNanStop;  // NaN residual: the loop condition ends the solve
      }
      s_flag = flag;
    }
    __syncthreads();
    if (s_flag) {
      if (blockIdx.x == 0 && tid == 0) {
        d.st->status = s_flag;
        d.st->halt = 1;
        if (s_flag == kIterCollapse) {
          d.st->ratio = gw[nsl].ratio;
          d.st->singular1 = gw[nsl].singular1;
        }
      }
      if (s_flag == kIterCollapse) return;
      // (NaN stop: the push itself succeeded; record it like the batched path)
      if (blockIdx.x == 0)
        for (int w = tid; w < (int)(sizeof(Gram) / 8); w += PS_NT)
          reinterpret_cast<uint64_t*>(d.grams + nsl)[w] = reinterpret_cast<const uint64_t*>(gw + nsl)[w];
      return;
    }
    if (blockIdx.x == 0) {
      for (int w = tid; w < (int)(sizeof(Gram) / 8); w += PS_NT)
        reinterpret_cast<uint64_t*>(d.grams + nsl)[w] = reinterpret_cast<const uint64_t*>(gw + nsl)[w];
      if (tid < S) {
        d.coef[cA(S) + tid] = sa[tid];
        d.coef[cNegA(S) + tid] = -sa[tid];
      }
    }
    if (t >= d.it_end) return;
  }
}

template <int S>
void run_persist(Ctx& c, const PersistDesc& d, int G, double bytes) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = G;
  cfg.blockDim = PS_NT;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  Launch lh(c, "somin_persist", bytes);
  CK(cudaLaunchKernelEx(&cfg, k_somin_persist<S>, d));
}

__global__ void k_any_nonzero(const double* x, int64_t n, int* flag) {
  SKC_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (x[i] != 0.0) {
      *flag = 1;
      return;
    }
}

}  // namespace

__global__ void k_flag_to_partial(const int* flag, double* partials) {
  SKC_PDL_ENTRY(); partials[0] = *flag ? 1.0 : 0.0; }

bool device_is_zero(Ctx& c, const double* x, int64_t n) {
  int* flag = (int*)c.workspace("is_zero_flag", sizeof(int));
  CK(cudaMemsetAsync(flag, 0, sizeof(int), c.stream));
  ++c.launches;
  launch_k(c, k_any_nonzero, std::min<int64_t>(1184, (n + 255) / 256), 256, 0, x, n, flag);
  CK(cudaGetLastError());
  double* p = (double*)c.workspace("is_zero_partial", sizeof(double) * kPartialPitch);
  launch_k(c, k_flag_to_partial, 1, 1, 0, flag, p);
  const int G = c.reduce_point(p, 1, 0, 1);  // across ranks: every rank sees every flag
  std::vector<double> h(G);
  CK(cudaMemcpyAsync(h.data(), p, sizeof(double) * G, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  for (double v : h)
    if (v != 0.0) return false;
  return true;
}

// K[j] = A^{j+1} src for j < J (krylov_pair's A R block, sstep.hpp:71-81): one matrix-powers
// sweep per at most mpk_max_depth levels for stencils, repeated applies for general CSR
static void powers(Ctx& c, const Op& op, const double* src, double* K, size_t np, int J, const int* halt) {
  const int maxj = powers_depth(c, op.d);
  if (maxj < 1) {
    for (int j = 0; j < J; ++j) {
      launch_apply(c, op.d, src, K + (size_t)j * np, halt, nullptr);
      src = K + (size_t)j * np;
    }
    return;
  }
  int done = 0;
  while (done < J) {
    const int d = std::min(J - done, maxj);
    double* outs[kMaxS + 1];
    outs[0] = nullptr;
    for (int j = 1; j <= d; ++j) outs[j] = K + (size_t)(done + j - 1) * np;
    launch_mpk(c, op.d, src, nullptr, outs, d, 0, nullptr, 1, nullptr, 0, halt, nullptr);
    src = K + (size_t)(done + d - 1) * np;
    done += d;
  }
}

// r = f - A x (x != 0) or r = f, plus the r.r partial at dot d0
static void initial_residual_dev(Ctx& c, const Op& op, const Geo& g, const double* f, const double* x, double* r,
                                 double* ax, bool x_zero, const double* coef, int ncoef, int idx_minus1,
                                 double* partials, int d0) {
  LinBuilder lb;
  if (!x_zero) {
    launch_apply(c, op.d, x, ax, nullptr, nullptr);
    lb.add_out(r, f);
    lb.add_term(ax, 1u, idx_minus1);  // r[i] -= ax[i] (solvers.hpp:65-66)
  } else {
    lb.add_out(r, f);
  }
  lb.add_dot(0, 0);
  lb.launch(c, g, coef, ncoef, partials, d0, nullptr, nullptr, "residual");
}

// ============================================================================ s-Omin
void somin_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep) {
  const bool gcr = cfg.unbounded_window;
  require(gcr || cfg.k >= 1, "s-omin: window k must be at least 1");
  validate_block_size(cfg, rep);
  const int s = (int)cfg.s;
  const int64_t n = op.n;
  const size_t np = pad_n(n);
  const Geo g = make_geo_for(c, op);
  rep.steady_iteration = gcr ? cfg.max_iterations + 1 : cfg.k;

  // window capacity (entries) and slot count
  const uint64_t kwin = gcr ? std::min<uint64_t>(cfg.max_iterations + 1, (uint64_t)kMaxWin - 1) : cfg.k;
  require(kwin <= (uint64_t)kMaxWin, "s-omin: window larger than the device scalar kernels support");
  const int nslot = (int)kwin + 1;

  // ---- workspace
  const size_t nvec = 2 + s + (size_t)nslot * 2 * s;  // r, ax, K[s], slots
  double* V = (double*)c.workspace("somin_vec", nvec * np * sizeof(double));
  double* r = V;
  double* ax = V + np;
  double* K = V + 2 * np;
  auto slot_p = [&](int sl, int col) { return V + (2 + s + (size_t)sl * 2 * s + col) * np; };
  auto slot_ap = [&](int sl, int col) { return V + (2 + s + (size_t)sl * 2 * s + s + col) * np; };
  // dot regions: W, m (one reduction point), then ||r||^2 directly followed by the C_e products,
  // so an s-step needs two reduction points across ranks
  const int dW = 0, dM = s * s, dRR = dM + s, dC = dRR + 1, dX = dC + (int)kwin * s * s;
  const int ndots = dX + (int)kwin * s * s;
  double* partials = (double*)c.workspace("somin_partials", (size_t)ndots * kPartialPitch * sizeof(double));
  const int ncoef = cB(s) + (int)kwin * s * s;
  double* coef = (double*)c.workspace("somin_coef", (size_t)ncoef * sizeof(double));
  double* scratch = (double*)c.workspace("somin_scratch", (size_t)(64 + 2 * kwin * s * s) * sizeof(double));
  Gram* grams = (Gram*)c.workspace("somin_grams", (size_t)nslot * sizeof(Gram));
  const uint64_t hcap = std::min<uint64_t>(cfg.max_iterations, 50000000ULL) + 2;
  double* hist = (double*)c.workspace("somin_hist", hcap * sizeof(double));
  SominState* st = (SominState*)c.workspace("somin_state", sizeof(SominState));
  {
    SominState h{};
    h.max_iter = (long long)cfg.max_iterations;
    h.fixed = cfg.fixed_steps ? 1 : 0;
    h.tol = cfg.tol;
    h.divf = cfg.divergence_factor;
    CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c.stream));
    double hc[cB(8) + 1];
    for (int i = 0; i < cB(s); ++i) hc[i] = 0.0;
    hc[cMinus1(s)] = -1.0;
    CK(cudaMemcpyAsync(coef, hc, sizeof(double) * cB(s), cudaMemcpyHostToDevice, c.stream));
  }
  const int* halt = &st->halt;

  // ---- initial residual (solvers.hpp:58-76) and setup (sstep.hpp:164-178)
  const bool x_zero = device_is_zero(c, x, n);
  initial_residual_dev(c, op, g, f, x, r, ax, x_zero, coef, ncoef, cMinus1(s), partials, dRR);
  launch_k(c, k_somin_start, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), dRR, 1), dRR);
  ++c.launches;
  CK(cudaGetLastError());
  // krylov_pair(r): P0 = [r, Ar, .., A^{s-1} r], AP0 = [Ar, .., A^s r]
  {
    powers(c, op, r, slot_ap(0, 0), np, s, halt);  // AP0 columns are consecutive
    LinBuilder lb;  // P0 columns are copies (krylov_block storage)
    lb.add_out(slot_p(0, 0), r);
    for (int j = 1; j < s; ++j) lb.add_out(slot_p(0, j), slot_ap(0, j - 1));
    lb.launch(c, g, coef, ncoef, partials, 0, halt, nullptr, "copy");
    std::vector<const double*> L, R;
    for (int j = 0; j < s; ++j) L.push_back(slot_ap(0, j));
    launch_gram_list(c, g, L, L, partials, dW, halt, nullptr, "gram_w");
    launch_gram_list(c, g, L, {r}, partials, dM, halt, nullptr, "gram_m");
    launch_k(c, k_somin_setup, 1, 256, 0, st, grams, coef, partials, c.reduce_point(partials, g.enc(), dW, s * s + s), dW, dM, s);
    ++c.launches;
    CK(cudaGetLastError());
  }

  // ---- iterations, enqueued in batches; host predicts the window deque
  std::vector<int> win{0};  // slot per window position
  std::vector<int> free_slots;
  for (int sl = nslot - 1; sl >= 1; --sl) free_slots.push_back(sl);
  SominState hs{};
  uint64_t enq = 0;
  const uint64_t batch = n <= (1 << 16) ? 32 : 8;
  bool gcr_full = false;
  CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  // small problems: whole iterations in one cooperative launch per chunk (see k_somin_persist)
  if (c.persist && !g.grouped() && op.d.kind != kIlu0 && !gcr && !cfg.debug_checks && c.world() == 1 && s <= 4 && cfg.k <= (uint64_t)PS_MAXK &&
      n <= (1 << 18)) {
    PersistDesc pd;
    std::memset(&pd, 0, sizeof pd);
    pd.op = op.d;
    pd.k = (int)cfg.k;
    pd.n = n;
    const int G = (int)std::min<int64_t>(c.sm_count, (n + PS_NT - 1) / PS_NT);
    pd.P = (n + G - 1) / G;
    pd.np = (int64_t)np;
    pd.x = x;
    pd.r = r;
    pd.K = K;
    pd.S0 = slot_p(0, 0);
    pd.partials = partials;
    pd.dRR = dRR;
    pd.dW = dW;
    pd.dC = dC;
    pd.grams = grams;
    pd.coef = coef;
    pd.st = st;
    pd.hist = hist;
    // algorithmic bytes of one iteration (profiling only): the batched path's operands
    const double bytes = 8.0 * (double)n * (3.0 * (double)cfg.k * s + 7.0 * s + 6.0);
    while (hs.status == kRunning && (uint64_t)hs.iters < cfg.max_iterations) {
      pd.it_end = hs.iters + 4096;
      switch (s) {
        case 1: run_persist<1>(c, pd, G, bytes); break;
        case 2: run_persist<2>(c, pd, G, bytes); break;
        case 3: run_persist<3>(c, pd, G, bytes); break;
        default: run_persist<4>(c, pd, G, bytes); break;
      }
      CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
      c.sync();
    }
    enq = cfg.max_iterations;
  }
  while (hs.status == kRunning && enq < cfg.max_iterations) {
    const uint64_t todo = std::min<uint64_t>(batch, cfg.max_iterations - enq);
    for (uint64_t it = 0; it < todo; ++it, ++enq) {
      const int cur = win.back();
      // x += P a ; r -= AP a ; ||r||^2   (sstep.hpp:183-193)
      {
        LinBuilder lb;
        lb.add_out(x, x);
        lb.add_out(r, r);
        for (int l = 0; l < s; ++l) lb.add_term(slot_p(cur, l), 1u, cA(s) + l);
        for (int l = 0; l < s; ++l) lb.add_term(slot_ap(cur, l), 2u, cNegA(s) + l - 1);
        lb.add_dot(1, 1);
        lb.launch(c, g, coef, ncoef, partials, dRR, halt, nullptr, "xr_update");
      }
      // across ranks the termination test on ||r|| runs after the C_e products below, sharing
      // their reduction point (the powers and products of the final iteration are spent for
      // nothing, once); on one GPU it runs here
      const bool pack_rr = c.world() > 1;
      if (!pack_rr) {
        launch_k(c, k_somin_norm, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), dRR, 1), dRR, hist);
        ++c.launches;
      }
      // krylov_pair(r) -> K[j] = A^{j+1} r  (matrix-powers sweep)
      powers(c, op, r, K, np, s, halt);
      // C_e = AP_e^T AR   (block_gram, sstep.hpp:207)
      Slots ws{};
      ws.n = (int)win.size();
      for (size_t e = 0; e < win.size(); ++e) ws.idx[e] = (int16_t)win[e];
      {
        std::vector<const double*> L, R;
        for (int sl : win)
          for (int l = 0; l < s; ++l) L.push_back(slot_ap(sl, l));
        for (int j = 0; j < s; ++j) R.push_back(K + (size_t)j * np);
        launch_gram_list(c, g, L, R, partials, dC, halt, nullptr, "gram_c");
      }
      if (pack_rr) {
        const int Grc = c.reduce_point(partials, g.enc(), dRR, 1 + ws.n * s * s);  // ||r||^2 and C_e together
        launch_k(c, k_somin_norm, 1, 256, 0, st, partials, Grc, dRR, hist);
        launch_k(c, k_somin_proj, 1, 256, 0, st, grams, ws, coef, partials, Grc, dC, s, scratch);
        c.launches += 2;
      } else {
        launch_k(c, k_somin_proj, 1, 256, 0, st, grams, ws, coef, partials, c.reduce_point(partials, g.enc(), dC, ws.n * s * s), dC, s, scratch);
        ++c.launches;
      }
      // new slot: P = R + sum_e P_e b_e ; AP = AR + sum_e AP_e b_e ; W ; m  (sstep.hpp:215-222)
      if (free_slots.empty()) {  // s-GCR window at the device limit
        gcr_full = true;
        break;
      }
      const int nsl = free_slots.back();
      free_slots.pop_back();
      if (2 * s <= 8) {  // one fused launch: P and AP halves share the powers block R / AR
        LinBuilder lb;
        for (int jc = 0; jc < s; ++jc) lb.add_out(slot_p(nsl, jc), jc == 0 ? r : K + (size_t)(jc - 1) * np);
        for (int jc = 0; jc < s; ++jc) lb.add_out(slot_ap(nsl, jc), K + (size_t)jc * np);
        const uint16_t lo = (uint16_t)((1u << s) - 1u), hi = (uint16_t)(lo << s);
        for (size_t e = 0; e < win.size(); ++e) {
          for (int l = 0; l < s; ++l) lb.add_term(slot_p(win[e], l), lo, cB(s) + (int)e * s * s + l * s);
          for (int l = 0; l < s; ++l) lb.add_term(slot_ap(win[e], l), hi, cB(s) + (int)e * s * s + l * s - s);
        }
        lb.add_extra(r);
        for (int a = 0; a < s; ++a)
          for (int b = a; b < s; ++b) lb.add_dot(s + a, s + b);
        for (int a = 0; a < s; ++a) lb.add_dot(s + a, 2 * s);
        lb.launch(c, g, coef, ncoef, partials, dW, halt, nullptr, "block_update");
      } else {
        // s > 4: the P half and the AP half as two launches of s outputs each.  One launch would
        // stage 2ks + s + 2 distinct vectors per point tile (s = 8: ~41) -- kilobyte-sized bulk
        // copies from that many streams and 2s accumulators per thread (measured 1.8 TB/s on C5);
        // the halves re-read the s - 1 shared powers once more but stream at the narrow rate.
        // Every output keeps its terms in the same order (same bits); W and m ride on the AP half.
        LinBuilder lp, la;
        for (int jc = 0; jc < s; ++jc) lp.add_out(slot_p(nsl, jc), jc == 0 ? r : K + (size_t)(jc - 1) * np);
        for (int jc = 0; jc < s; ++jc) la.add_out(slot_ap(nsl, jc), K + (size_t)jc * np);
        const uint16_t all = (uint16_t)((1u << s) - 1u);
        for (size_t e = 0; e < win.size(); ++e) {
          for (int l = 0; l < s; ++l) lp.add_term(slot_p(win[e], l), all, cB(s) + (int)e * s * s + l * s);
          for (int l = 0; l < s; ++l) la.add_term(slot_ap(win[e], l), all, cB(s) + (int)e * s * s + l * s);
        }
        la.add_extra(r);
        for (int a = 0; a < s; ++a)
          for (int b = a; b < s; ++b) la.add_dot(a, b);
        for (int a = 0; a < s; ++a) la.add_dot(a, s);
        lp.launch(c, g, coef, ncoef, partials, dW, halt, nullptr, "block_update");
        la.launch(c, g, coef, ncoef, partials, dW, halt, nullptr, "block_update");
      }
      if (cfg.debug_checks) {
        std::vector<const double*> L, R;
        for (int sl : win)
          for (int l = 0; l < s; ++l) L.push_back(slot_ap(sl, l));
        for (int j = 0; j < s; ++j) R.push_back(slot_ap(nsl, j));
        launch_gram_list(c, g, L, R, partials, dX, halt, nullptr, "gram_debug");
      }
      int Gp = c.reduce_point(partials, g.enc(), dW, s * (s + 1) / 2 + s);
      if (cfg.debug_checks) Gp = c.reduce_point(partials, g.enc(), dX, ws.n * s * s);
      launch_k(c, k_somin_push, 1, 256, 0, st, grams, nsl, coef, partials, Gp, dW, dW + s * (s + 1) / 2, s, cfg.debug_checks ? 1 : 0, ws, dX, scratch);
      ++c.launches;
      CK(cudaGetLastError());
      // deque bookkeeping (sstep.hpp:235-237)
      win.push_back(nsl);
      if (!gcr && win.size() > cfg.k) {
        free_slots.push_back(win.front());
        win.erase(win.begin());
      }
    }
    CK(cudaMemcpyAsync(&hs, st, sizeof hs, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (gcr_full && hs.status == kRunning)
      fail(SKC_EINVAL, "s-gcr: window exceeds the device limit of " + std::to_string(kMaxWin) + " blocks");
  }

  // ---- rebuild the report by replaying the reference control flow
  std::vector<double> h(hs.iters + 1, 0.0);
  if (hs.iters > 0)
    CK(cudaMemcpy(h.data() + 1, hist + 1, sizeof(double) * hs.iters, cudaMemcpyDeviceToHost));
  skc_op_counter& cnt = rep.op_counts;
  if (!x_zero) add(cnt, 0, 1, 1);
  cnt.termination_dots += 1;
  rep.history.push_back(hs.r0n);
  double rn = hs.r0n;
  uint64_t peak = 0;
  if (rn > cfg.tol) {
    add(cnt, (uint64_t)s * (s + 1) / 2, (uint64_t)s, 0);
    if (hs.status == kSetupCollapse) {
      rep.breakdown = "basis collapse at setup (" + gram_message(hs.singular1, hs.ratio) + ")";
      rep.op_history.push_back(cnt);
      rep.converged = false;
      rep.final_residual = rn;
      return;
    }
    peak = 1;
  }
  rep.op_history.push_back(cnt);
  uint64_t nwin = peak;
  for (long long t = 1; t <= hs.iters; ++t) {
    add(cnt, (uint64_t)s, 0, 2ULL * s);
    cnt.termination_dots += 1;
    rep.iterations = (uint64_t)t;
    rn = h[t];
    rep.history.push_back(rn);
    const bool last = t == hs.iters;
    if (last && (hs.status == kConverged || hs.status == kMaxIter)) break;
    if (last && hs.status == kDiverged) {
      rep.breakdown = "divergence: residual grew beyond " + fmt_double(cfg.divergence_factor) + "x the initial norm";
      break;
    }
    add(cnt, nwin * s * s + (uint64_t)s * (s + 1) / 2, (uint64_t)s, nwin * 2ULL * s * s);
    if (last && hs.status == kLogic) fail(SKC_ELOGIC, "s-omin: block A-direction orthogonality lost");
    if (last && hs.status == kIterCollapse) {
      rep.breakdown = "basis collapse at iteration " + std::to_string(t) + " (" +
                      gram_message(hs.singular1, hs.ratio) + ")";
      break;
    }
    ++nwin;
    peak = std::max(peak, nwin);
    if (!gcr && nwin > cfg.k) --nwin;
    rep.op_history.push_back(cnt);
  }
  cnt.stored_vectors = 2 + 2ULL * s * peak;
  rep.converged = rn <= cfg.tol;
  rep.final_residual = rep.history.back();
}

// ============================================================================ s-MR
namespace {

struct SmrState {
  int status, halt, singular1, pad;
  long long iters, max_iter;
  double tol, rn, ratio;
};

__global__ void k_smr_start(SmrState* st, const double* partials, int G, int d0, double* hist) {
  SKC_PDL_ENTRY();
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    const double rn = sqrt(v[0]);
    st->rn = rn;
    hist[0] = rn;
    if (!(rn > st->tol) || st->iters >= st->max_iter) {
      st->status = kConverged;
      st->halt = 1;
    }
  }
}

// W = gram_self(AR), m = AR^T r, a = W^{-1} m (sstep.hpp:96-101)
__global__ void k_smr_solve(SmrState* st, double* coef, const double* partials, int G, int dW, int dm, int s) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[kMaxS * kMaxS + kMaxS];
  reduce_dots_dev(partials, G, dW, s * s, v);
  reduce_dots_dev(partials, G, dm, s, v + s * s);
  if (threadIdx.x == 0) {
    double W[kMaxS * kMaxS];
    for (int q = 0; q < s * s; ++q) W[q] = v[q];
    for (int j = 0; j < s; ++j)
      for (int l = j + 1; l < s; ++l) {
        const double avg = (W[j * s + l] + W[l * s + j]) / 2.0;
        W[j * s + l] = avg;
        W[l * s + j] = avg;
      }
    Gram gm;
    gram_factor_dev(gm, W, s);
    if (!gm.ok) {
      st->status = kIterCollapse;
      st->halt = 1;
      st->ratio = gm.ratio;
      st->singular1 = gm.singular1;
      return;
    }
    double a[kMaxS];
    gram_solve_dev(gm, v + s * s, a);
    for (int l = 0; l < s; ++l) {
      coef[l] = a[l];
      coef[s + l] = -a[l];
    }
  }
}

__global__ void k_smr_norm(SmrState* st, const double* partials, int G, int d0, double* hist) {
  SKC_PDL_ENTRY();
  if (st->halt) return;
  __shared__ double v[1];
  reduce_dots_dev(partials, G, d0, 1, v);
  if (threadIdx.x == 0) {
    const double rn = sqrt(v[0]);
    st->rn = rn;
    st->iters += 1;
    hist[st->iters] = rn;
    if (!(rn > st->tol) || st->iters >= st->max_iter) {
      st->status = kConverged;
      st->halt = 1;
    }
  }
}

}  // namespace

// one s-MR step on device buffers x, r (halt-guarded); K holds s vectors
static void smr_step_enqueue(Ctx& c, const Op& op, const Geo& g, double* x, double* r, double* K, size_t np, int s,
                             double* coef, int ncoef, double* partials, SmrState* st, double* hist) {
  const int* halt = &st->halt;
  powers(c, op, r, K, np, s, halt);
  std::vector<const double*> AR;
  for (int j = 0; j < s; ++j) AR.push_back(K + (size_t)j * np);
  launch_gram_list(c, g, AR, AR, partials, 1, halt, nullptr, "gram_w");
  launch_gram_list(c, g, AR, {r}, partials, 1 + s * s, halt, nullptr, "gram_m");
  launch_k(c, k_smr_solve, 1, 256, 0, st, coef, partials, c.reduce_point(partials, g.enc(), 1, s * s + s), 1, 1 + s * s, s);
  ++c.launches;
  // x += R a (R = [r, A r, .., A^{s-1} r]); r -= AR a  (sstep.hpp:102-103)
  LinBuilder lb;
  lb.add_out(x, x);
  lb.add_out(r, r);
  lb.add_term(r, 1u, 0);
  for (int l = 1; l < s; ++l) lb.add_term(K + (size_t)(l - 1) * np, 1u, l);
  for (int l = 0; l < s; ++l) lb.add_term(K + (size_t)l * np, 2u, s + l - 1);
  lb.add_dot(1, 1);
  lb.launch(c, g, coef, ncoef, partials, 0, halt, nullptr, "xr_update");
  launch_k(c, k_smr_norm, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), 0, 1), 0, hist);
  ++c.launches;
  CK(cudaGetLastError());
}

void smr_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep) {
  validate_block_size(cfg, rep);
  const int s = (int)cfg.s;
  const int64_t n = op.n;
  const size_t np = pad_n(n);
  const Geo g = make_geo_for(c, op);
  double* V = (double*)c.workspace("smr_vec", (2 + (size_t)s) * np * sizeof(double));
  double *r = V, *ax = V + np, *K = V + 2 * np;
  const int ncoef = 2 * s + 1;
  double* coef = (double*)c.workspace("smr_coef", ncoef * sizeof(double));
  double* partials = (double*)c.workspace("smr_partials", (size_t)(1 + s * s + s) * kPartialPitch * sizeof(double));
  const uint64_t hcap = std::min<uint64_t>(cfg.max_iterations, 50000000ULL) + 2;
  double* hist = (double*)c.workspace("smr_hist", hcap * sizeof(double));
  SmrState* st = (SmrState*)c.workspace("smr_state", sizeof(SmrState));
  SmrState h{};
  h.max_iter = (long long)cfg.max_iterations;
  h.tol = cfg.tol;
  CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c.stream));
  {
    double hc[17] = {0};
    hc[2 * s] = -1.0;
    CK(cudaMemcpyAsync(coef, hc, sizeof(double) * ncoef, cudaMemcpyHostToDevice, c.stream));
  }
  const bool x_zero = device_is_zero(c, x, n);
  initial_residual_dev(c, op, g, f, x, r, ax, x_zero, coef, ncoef, 2 * s, partials, 0);
  launch_k(c, k_smr_start, 1, 256, 0, st, partials, c.reduce_point(partials, g.enc(), 0, 1), 0, hist);
  ++c.launches;
  uint64_t enq = 0;
  const uint64_t batch = n <= (1 << 16) ? 32 : 8;
  CK(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  while (!h.halt && enq < cfg.max_iterations) {
    const uint64_t todo = std::min<uint64_t>(batch, cfg.max_iterations - enq);
    for (uint64_t it = 0; it < todo; ++it, ++enq)
      smr_step_enqueue(c, op, g, x, r, K, np, s, coef, ncoef, partials, st, hist);
    CK(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
  }
  // replay (sstep.hpp:109-135)
  std::vector<double> hh(h.iters + 1);
  CK(cudaMemcpy(hh.data(), hist, sizeof(double) * (h.iters + 1), cudaMemcpyDeviceToHost));
  skc_op_counter& cnt = rep.op_counts;
  if (!x_zero) add(cnt, 0, 1, 1);
  cnt.termination_dots += 1;
  rep.history.push_back(hh[0]);
  cnt.stored_vectors = 2 + 2ULL * s;
  rep.op_history.push_back(cnt);
  double rn = hh[0];
  for (long long t = 1; t <= h.iters; ++t) {
    add(cnt, (uint64_t)s * (s + 1) / 2 + s, (uint64_t)s, 2ULL * s);
    cnt.termination_dots += 1;
    rep.iterations = t;
    rn = hh[t];
    rep.history.push_back(rn);
    rep.op_history.push_back(cnt);
  }
  if (h.status == kIterCollapse) {
    add(cnt, (uint64_t)s * (s + 1) / 2 + s, (uint64_t)s, 0);
    rep.breakdown = "basis collapse at iteration " + std::to_string(h.iters) + " (" +
                    gram_message(h.singular1, h.ratio) + "); reduce s";
  }
  rep.converged = rn <= cfg.tol;
  rep.final_residual = rep.history.back();
}

void smr_step_device(Ctx& c, const Op& op, double* x, double* r, uint64_t s64, double* coeffs,
                     skc_op_counter* counter) {
  require(s64 >= 1, "smr_step: s must be at least 1");
  require(s64 <= (uint64_t)kMaxS, "smr_step: s above the supported block width 8");
  const int s = (int)s64;
  const int64_t n = op.n;
  const size_t np = pad_n(n);
  const Geo g = make_geo_for(c, op);
  double* K = (double*)c.workspace("smr_vec", (2 + (size_t)s) * np * sizeof(double)) + 2 * np;
  const int ncoef = 2 * s + 1;
  double* coef = (double*)c.workspace("smr_coef", ncoef * sizeof(double));
  double* partials = (double*)c.workspace("smr_partials", (size_t)(1 + s * s + s) * kPartialPitch * sizeof(double));
  double* hist = (double*)c.workspace("smr_hist", 4 * sizeof(double));
  SmrState* st = (SmrState*)c.workspace("smr_state", sizeof(SmrState));
  SmrState h{};
  h.max_iter = 1;
  h.tol = -1.0;
  CK(cudaMemcpyAsync(st, &h, sizeof h, cudaMemcpyHostToDevice, c.stream));
  smr_step_enqueue(c, op, g, x, r, K, np, s, coef, ncoef, partials, st, hist);
  CK(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  double a[kMaxS];
  CK(cudaMemcpyAsync(a, coef, sizeof(double) * s, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (h.status == kIterCollapse) fail(SKC_EBREAKDOWN, gram_message(h.singular1, h.ratio));
  if (coeffs) std::memcpy(coeffs, a, sizeof(double) * s);
  if (counter) {
    add(*counter, (uint64_t)s * (s + 1) / 2 + s, (uint64_t)s, 2ULL * s);
  }
}

}  // namespace skc
