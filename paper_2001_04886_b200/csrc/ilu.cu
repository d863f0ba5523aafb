// ilu.cu -- ILU(0) right preconditioning on the device: the operator A (LU)^{-1}
// (right_preconditioned, ilu0.hpp:138-146) and the solve z = (LU)^{-1} r (ilu0_apply,
// ilu0.hpp:99-127), the pieces the reference driver composes when `precondition` is set
// (solve_linear, bench.hpp:149-191).
//
// The factorization is the reference's row-wise IKJ elimination restricted to pattern(A)
// (ilu0_factor, ilu0.hpp:45-95), run on the device: row i only reads the finished rows of its
// lower neighbours, so the rows are walked in the level schedule of L (a barrier between
// levels) and every row is eliminated by one thread in the reference's order -- its lower
// entries by ascending column, each subtracting mult * U(k, :) from the matching entries, the
// same IEEE operations (no contraction), hence the same bits.  The reference's error behaviour:
// a row without a diagonal is an invalid argument (checked on the host with the pattern), a
// pivot below 1e-14 max|diag(A)| a breakdown naming the first such row.
//
// The triangular solves are level-scheduled: rows are grouped by their dependency depth in L
// (resp. U), and one cooperative launch walks the levels with a grid barrier between them,
// every row of a level on its own thread.  Each row is evaluated exactly as the reference's
// sequential loop does (acc -= l * z in the row's column order, then / diag for U), so the
// result is bit-identical to ilu0_apply; only the order in which independent rows are
// visited changes.  For a 5-point grid in natural order the levels are the anti-diagonals
// (nx + ny - 1 of them).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "device_util.cuh"
#include "skc_internal.hpp"

namespace skc {

namespace {

constexpr int TR_NT = 512;

// One CTA walks every level with a block barrier between them (no grid barrier): used when the
// widest level fits the CTA a few times over, e.g. the anti-diagonals of a 2D grid, where the
// solve is a chain of nx + ny - 1 short levels and the cost is the per-level latency
constexpr int TR1_NT = 1024;
template <bool LOWER>
__global__ void __launch_bounds__(TR1_NT) k_trsv1(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                  const double* __restrict__ v, const int32_t* __restrict__ perm,
                                                  const int64_t* __restrict__ lev, int nlev, const double* r, double* z,
                                                  const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  for (int L = 0; L < nlev; ++L) {
    const int64_t e = lev[L + 1];
    for (int64_t q = lev[L] + threadIdx.x; q < e; q += TR1_NT) {
      const int i = perm[q];
      if (LOWER) {
        double acc = r[i];
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) acc = __dsub_rn(acc, __dmul_rn(v[p], z[ci[p]]));
        z[i] = acc;
      } else {
        double acc = z[i], dia = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          if (ci[p] == i)
            dia = v[p];
          else
            acc = __dsub_rn(acc, __dmul_rn(v[p], z[ci[p]]));
        }
        z[i] = __ddiv_rn(acc, dia);
      }
    }
    __syncthreads();
  }
}

template <bool LOWER>
__global__ void __launch_bounds__(TR_NT) k_trsv(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                const double* __restrict__ v, const int32_t* __restrict__ perm,
                                                const int64_t* __restrict__ lev, int nlev, const double* r, double* z,
                                                const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gn = (int64_t)gridDim.x * blockDim.x;
  for (int L = 0; L < nlev; ++L) {
    const int64_t e = lev[L + 1];
    for (int64_t q = lev[L] + gt; q < e; q += gn) {
      const int i = perm[q];
      if (LOWER) {  // unit lower: z_i = r_i - sum_j l_ij z_j
        double acc = r[i];
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) acc = __dsub_rn(acc, __dmul_rn(v[p], z[ci[p]]));
        z[i] = acc;
      } else {  // upper: z_i = (z_i - sum_{j>i} u_ij z_j) / u_ii
        double acc = z[i], dia = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          if (ci[p] == i)
            dia = v[p];
          else
            acc = __dsub_rn(acc, __dmul_rn(v[p], z[ci[p]]));
        }
        z[i] = __ddiv_rn(acc, dia);
      }
    }
    if (L + 1 < nlev) grid.sync();
  }
}

// Strip wavefront for a 2D 5-point grid in natural order (L: S and W neighbours; U: E and N).
// One warp per 32-column strip; lane k takes column k of the strip (mirrored for U) and, at
// step t, row t - k (descending rows for U): its in-row neighbour (W / E) is the value lane
// k-1 produced one step earlier (a shuffle), its cross-row neighbour (S / N) its own previous
// value, so the 32 lanes advance along an anti-diagonal with no barrier.  Lane 0's in-row
// neighbour belongs to the adjacent strip (left for L, right for U): that strip publishes
// rows-done counters (release, every 32 rows) and this one fetches the neighbour column 32
// rows at a time (acquire).  The strip's own operands are prefetched 8 steps ahead.  Every
// row is the reference's sequential evaluation (ilu0_apply: acc -= l * z in column order,
// then / diag for U), so z is bit-identical to the level-scheduled solve.
#ifndef SKC_SW_D
#define SKC_SW_D 16
#endif
constexpr int SW_D = SKC_SW_D;
constexpr unsigned long long kBndSentinel = 0x7FF0DEADBEEF0001ULL;  // signalling NaN

__global__ void k_fill_bits(double* p, unsigned long long bits, int64_t n) {
  SKC_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<unsigned long long*>(p)[i] = bits;
}
template <bool LOWER>
__global__ void __launch_bounds__(32) k_trsv_strip(const double* __restrict__ a1, const double* __restrict__ a2,
                                                   const double* __restrict__ ac, const uint8_t* __restrict__ msk,
                                                   int nx, int ny, const double* r, double* z, double* bnd,
                                                   int* stalled, const int* halt, const int* cond) {
  SKC_PDL_ENTRY();
  if (skip_launch(halt, cond)) return;
  const int k = threadIdx.x, sx = blockIdx.x, nstrip = gridDim.x;
  const int x = LOWER ? 32 * sx + k : 32 * sx + 31 - k;
  const bool col_ok = x < nx;
  const int nb = LOWER ? sx - 1 : sx + 1;  // the strip owning lane 0's in-row neighbour
  const bool has_nb = nb >= 0 && nb < nstrip;
  const int xn = LOWER ? 32 * sx - 1 : 32 * sx + 32;  // lane 0's in-row neighbour column
  // the lane that owns the column the next strip needs (x = 32 sx + 31 for L, 32 sx for U)
  const bool publisher = k == 31;
  auto row_of = [&](int t) { return LOWER ? t - k : ny - 1 - (t - k); };
  double zlast = 0.0, wchunk = 0.0;
  // operand ring: (in-row coefficient, cross-row coefficient, diagonal / rhs, mask)
  double q1[SW_D], q2[SW_D], qc[SW_D], qz[SW_D];
  uint8_t qm[SW_D];
  auto fetch = [&](int t, int u) {
    const int y = row_of(t);
    const bool ok = col_ok && t - k >= 0 && t - k < ny;
    const int64_t p = (int64_t)(ok ? y : 0) * nx + (ok ? x : 0);
    q1[u] = ok ? a1[p] : 0.0;
    q2[u] = ok ? a2[p] : 0.0;
    qc[u] = ok ? (LOWER ? r[p] : ac[p]) : 0.0;
    qz[u] = !LOWER && ok ? z[p] : 0.0;  // (U: the forward solve's value, rewritten only by this lane)
    qm[u] = ok ? msk[p] : 0;
  };
#pragma unroll
  for (int u = 0; u < SW_D; ++u) fetch(u, u);
  const int T = ny + 31;
  for (int t0 = 0; t0 < T; t0 += SW_D) {
#pragma unroll
    for (int u = 0; u < SW_D; ++u) {
      const int t = t0 + u;
      if (t >= T) break;
      if ((t & 31) == 0 && has_nb) {  // lane 0's in-row neighbours for rows t .. t+31
        // each lane waits for its row's value in the neighbour strip's boundary column to
        // replace the sentinel (a signalling NaN, which arithmetic never produces), bounded
        double w = 0.0;
        if (t + k < ny) {
          const volatile unsigned long long* b =
              reinterpret_cast<const volatile unsigned long long*>(bnd + (int64_t)nb * ny + t + k);
          unsigned long long bits = *b;
          for (int spin = 0; bits == kBndSentinel && spin < (1 << 26); ++spin) bits = *b;
          if (bits == kBndSentinel) {  // the neighbour strip never delivered: flag it (the host raises)
            atomicExch(stalled, 1);
            bits = 0;
          }
          w = __longlong_as_double((long long)bits);
        }
        wchunk = w;
      }
      const double from_prev_lane = __shfl_up_sync(0xffffffffu, zlast, 1);
      const double nbv = __shfl_sync(0xffffffffu, wchunk, t & 31);
      const double in_row = k == 0 ? nbv : from_prev_lane;
      const int y = row_of(t);
      const bool active = col_ok && t - k >= 0 && t - k < ny;
      if (active) {
        const int64_t p = (int64_t)y * nx + x;
        double acc;
        if (LOWER) {  // acc = r - l_S z_S - l_W z_W  (columns p - nx, p - 1)
          acc = qc[u];
          if (qm[u] & 1) acc = __dsub_rn(acc, __dmul_rn(q2[u], zlast));
          if (qm[u] & 2) acc = __dsub_rn(acc, __dmul_rn(q1[u], in_row));
        } else {      // acc = (z - u_E z_E - u_N z_N) / u_C  (columns p + 1, p + nx)
          acc = qz[u];
          if (qm[u] & 1) acc = __dsub_rn(acc, __dmul_rn(q1[u], in_row));
          if (qm[u] & 2) acc = __dsub_rn(acc, __dmul_rn(q2[u], zlast));
          acc = __ddiv_rn(acc, qc[u]);
        }
        z[p] = acc;
        zlast = acc;
        const int done = t - k + 1;  // rows of this column finished
        if (publisher) *reinterpret_cast<volatile double*>(bnd + (int64_t)sx * ny + (done - 1)) = acc;
      }
      fetch(t + SW_D, u);
    }
  }
}

template <bool LOWER>
void launch_trsv(Ctx& c, const IluData& d, const double* r, double* z, const int* halt, const int* cond) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = c.sm_count;
  cfg.blockDim = TR_NT;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const double bytes = LOWER ? 8.0 * (2.0 * d.n) + 12.0 * d.nnz_l + 12.0 * d.n : 8.0 * (2.0 * d.n) + 12.0 * d.nnz_u + 12.0 * d.n;
  Launch lh(c, LOWER ? "ilu_lower" : "ilu_upper", bytes);
  // the strips wait on each other, so every strip must be resident at once: use them only when
  // the cooperative grid fits (and the grid has rows to pipeline; a 1D ny = 1 "grid" is serial)
  const int ns = d.gnx > 0 ? (int)((d.gnx + 31) / 32) : 0;
  bool strips = d.gnx > 0 && d.gny > 1 && c.ilu_strips;
  if (strips) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trsv_strip<LOWER>, 32, 0));
    strips = (int64_t)ns <= (int64_t)per_sm * c.sm_count;
  }
  if (strips) {
    double* bnd = d.bnd;
    launch_k(c, k_fill_bits, (unsigned)std::min<int64_t>(1184, (ns * d.gny + 255) / 256), 256, 0, bnd, kBndSentinel,
             (int64_t)ns * d.gny);
    ++c.launches;
    cudaLaunchConfig_t sc{};
    sc.gridDim = ns;
    sc.blockDim = 32;
    sc.stream = c.stream;
    cudaLaunchAttribute sa[1];
    sa[0].id = cudaLaunchAttributeCooperative;  // (all strips resident: they wait on each other)
    sa[0].val.cooperative = 1;
    sc.attrs = sa;
    sc.numAttrs = 1;
    if (LOWER)
      CK(cudaLaunchKernelEx(&sc, k_trsv_strip<true>, d.lW, d.lS, (const double*)nullptr, d.lm, (int)d.gnx, (int)d.gny,
                            r, z, bnd, d.stalled, halt, cond));
    else
      CK(cudaLaunchKernelEx(&sc, k_trsv_strip<false>, d.uE, d.uN, d.uC, d.um, (int)d.gnx, (int)d.gny,
                            (const double*)nullptr, z, bnd, d.stalled, halt, cond));
    return;
  }
  if ((LOWER ? d.maxw_l : d.maxw_u) <= 8 * TR1_NT) {
    if (LOWER)
      launch_k(c, k_trsv1<true>, 1, TR1_NT, 0, d.lrp, d.lci, d.lv, d.lperm, d.llev, d.nlev_l, r, z, halt, cond);
    else
      launch_k(c, k_trsv1<false>, 1, TR1_NT, 0, d.urp, d.uci, d.uv, d.uperm, d.ulev, d.nlev_u, (const double*)nullptr, z,
               halt, cond);
    return;
  }
  if (LOWER)
    CK(cudaLaunchKernelEx(&cfg, k_trsv<true>, d.lrp, d.lci, d.lv, d.lperm, d.llev, d.nlev_l, r, z, halt, cond));
  else
    CK(cudaLaunchKernelEx(&cfg, k_trsv<false>, d.urp, d.uci, d.uv, d.uperm, d.ulev, d.nlev_u, (const double*)nullptr, z,
                          halt, cond));
}

template <class T>
const T* upload(Op& owner, const std::vector<T>& h) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(sizeof(T) * h.size(), 16)));
  owner.owned.push_back(p);
  if (!h.empty()) CK(cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return static_cast<const T*>(p);
}

// rows grouped by level (ascending row within a level); levels from the dependency depth
void level_schedule(int64_t n, const std::vector<int64_t>& rp, const std::vector<int32_t>& ci, bool lower,
                    std::vector<int32_t>& perm, std::vector<int64_t>& lev) {
  std::vector<int32_t> depth(n, 0);
  int32_t maxd = 0;
  auto row = [&](int64_t i) {
    int32_t dd = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] != i) dd = std::max(dd, depth[ci[p]] + 1);
    depth[i] = dd;
    maxd = std::max(maxd, dd);
  };
  if (lower)
    for (int64_t i = 0; i < n; ++i) row(i);
  else
    for (int64_t i = n - 1; i >= 0; --i) row(i);
  lev.assign((size_t)maxd + 2, 0);
  for (int64_t i = 0; i < n; ++i) ++lev[(size_t)depth[i] + 1];
  for (size_t k = 1; k < lev.size(); ++k) lev[k] += lev[k - 1];
  perm.assign(n, 0);
  std::vector<int64_t> fill(lev.begin(), lev.end() - 1);
  for (int64_t i = 0; i < n; ++i) perm[fill[depth[i]]++] = (int32_t)i;
}

}  // namespace

namespace {

// row i of ilu0_factor (ilu0.hpp:59-90): lu holds A's values on entry and the factor on exit;
// the rows it reads (its lower neighbours k) are finished.  Loads bypass L1 (rows finished by
// other CTAs before the last grid barrier).
__device__ __forceinline__ void ilu_factor_row(int i, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                               const int64_t* __restrict__ dg, double* lu, double floor_, int* fail) {
  const int64_t b = rp[i], e = rp[i + 1];
  for (int64_t p = b; p < e && ci[p] < i; ++p) {
    const int k = ci[p];
    const int64_t dk = dg[k];
    const double mult = __ddiv_rn(__ldcg(lu + p), __ldcg(lu + dk));
    lu[p] = mult;
    int64_t w = p + 1;  // row i's columns above k, merged with row k's columns above its diagonal
    const int64_t ke = rp[k + 1];
    for (int64_t q = dk + 1; q < ke; ++q) {
      const int c = ci[q];
      while (w < e && ci[w] < c) ++w;
      if (w < e && ci[w] == c) lu[w] = __dsub_rn(__ldcg(lu + w), __dmul_rn(mult, __ldcg(lu + q)));
    }
  }
  if (fabs(__ldcg(lu + dg[i])) < floor_) atomicMin(fail, i);
}

// every level in one CTA (narrow levels, e.g. the anti-diagonals of a 2D grid)
__global__ void __launch_bounds__(1024) k_ilu_factor1(const int64_t* rp, const int32_t* ci, const int64_t* dg,
                                                       const int32_t* perm, const int64_t* lev, int nlev, double* lu,
                                                       double floor_, int* fail) {
  for (int L = 0; L < nlev; ++L) {
    for (int64_t q = lev[L] + threadIdx.x; q < lev[L + 1]; q += blockDim.x) ilu_factor_row(perm[q], rp, ci, dg, lu, floor_, fail);
    __syncthreads();
  }
}

// wide levels: one cooperative grid, a grid barrier between levels
__global__ void k_ilu_factor(const int64_t* rp, const int32_t* ci, const int64_t* dg, const int32_t* perm,
                             const int64_t* lev, int nlev, double* lu, double floor_, int* fail) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int L = 0; L < nlev; ++L) {
    for (int64_t q = lev[L] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < lev[L + 1]; q += stride)
      ilu_factor_row(perm[q], rp, ci, dg, lu, floor_, fail);
    grid.sync();
  }
}

}  // namespace

// ilu0_factor (ilu0.hpp:45-95) on the device: the factor values in A's pattern, returned to the
// host (lu).  The host checks the pattern (a diagonal in every row) and max|diag(A)|.
void ilu0_factor_device(Ctx& c, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals,
                        std::vector<double>& lu) {
  const int64_t nnz = n ? (int64_t)offs[n] : 0;
  lu.assign(vals, vals + nnz);
  if (n == 0) return;
  std::vector<int64_t> rp(offs, offs + n + 1), dg(n);
  std::vector<int32_t> ci(nnz);
  double max_diag = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    bool found = false;
    for (uint64_t p = offs[i]; p < offs[i + 1]; ++p) {
      ci[p] = (int32_t)cols[p];
      if (cols[p] == (uint64_t)i) {
        dg[i] = (int64_t)p;
        found = true;
        max_diag = std::max(max_diag, std::abs(vals[p]));
      }
    }
    require(found, "ilu0: row " + std::to_string(i + 1) + " has no diagonal entry");
  }
  // level schedule of the lower pattern (rows grouped by elimination depth)
  std::vector<int64_t> lrp(n + 1, 0);
  std::vector<int32_t> lci;
  for (int64_t i = 0; i < n; ++i) {
    for (uint64_t p = offs[i]; p < offs[i + 1] && cols[p] < (uint64_t)i; ++p) lci.push_back((int32_t)cols[p]);
    lrp[i + 1] = (int64_t)lci.size();
  }
  std::vector<int32_t> perm;
  std::vector<int64_t> lev;
  level_schedule(n, lrp, lci, true, perm, lev);
  int64_t maxw = 0;
  for (size_t q = 0; q + 1 < lev.size(); ++q) maxw = std::max(maxw, lev[q + 1] - lev[q]);
  const int nlev = (int)lev.size() - 1;
  // device buffers: one allocation
  const size_t b_rp = sizeof(int64_t) * (n + 1), b_dg = sizeof(int64_t) * n, b_lev = sizeof(int64_t) * lev.size();
  const size_t b_ci = sizeof(int32_t) * std::max<int64_t>(nnz, 1), b_pm = sizeof(int32_t) * n, b_lu = sizeof(double) * std::max<int64_t>(nnz, 1);
  char* buf = (char*)c.workspace("ilu_factor", b_rp + b_dg + b_lev + b_lu + b_ci + b_pm + 16);
  int64_t* d_rp = (int64_t*)buf;
  int64_t* d_dg = (int64_t*)(buf + b_rp);
  int64_t* d_lev = (int64_t*)(buf + b_rp + b_dg);
  double* d_lu = (double*)(buf + b_rp + b_dg + b_lev);
  int32_t* d_ci = (int32_t*)(buf + b_rp + b_dg + b_lev + b_lu);
  int32_t* d_pm = (int32_t*)((char*)d_ci + b_ci);
  int* d_fail = (int*)((char*)d_pm + b_pm);
  CK(cudaMemcpyAsync(d_rp, rp.data(), b_rp, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(d_dg, dg.data(), b_dg, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(d_lev, lev.data(), b_lev, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(d_lu, lu.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(d_ci, ci.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(d_pm, perm.data(), b_pm, cudaMemcpyHostToDevice, c.stream));
  const int no_fail = 0x7fffffff;
  CK(cudaMemcpyAsync(d_fail, &no_fail, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  const double floor_ = 1e-14 * max_diag;
  {
    Launch lh(c, "ilu_factor", 8.0 * 3.0 * (double)nnz);
    if (maxw <= 8 * 1024) {
      k_ilu_factor1<<<1, 1024, 0, c.stream>>>(d_rp, d_ci, d_dg, d_pm, d_lev, nlev, d_lu, floor_, d_fail);
      CK(cudaGetLastError());
    } else {
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilu_factor, 256, 0));
      const int G = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * c.sm_count, (maxw + 255) / 256));
      void* args[] = {&d_rp, &d_ci, &d_dg, &d_pm, &d_lev, (void*)&nlev, &d_lu, (void*)&floor_, &d_fail};
      CK(cudaLaunchCooperativeKernel((void*)k_ilu_factor, G, 256, args, 0, c.stream));
    }
  }
  int fail = no_fail;
  CK(cudaMemcpyAsync(&fail, d_fail, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaMemcpyAsync(lu.data(), d_lu, sizeof(double) * nnz, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (fail != no_fail) skc::fail(SKC_EBREAKDOWN, "ilu0: zero pivot at row " + std::to_string(fail + 1));
}

void build_ilu0_op(Ctx& c, Op& op, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals) {
  op.ilu = std::make_unique<IluData>();
  IluData& d = *op.ilu;
  build_csr_op(c, d.base, n, offs, cols, vals);  // validates the CSR invariants; one GPU only
  std::vector<double> lu;
  ilu0_factor_device(c, n, offs, cols, vals, lu);
  // split into L (strictly lower) and U (diagonal and above), A's column order kept
  std::vector<int64_t> lrp(n + 1, 0), urp(n + 1, 0);
  std::vector<int32_t> lci, uci;
  std::vector<double> lv, uv;
  for (int64_t i = 0; i < n; ++i) {
    for (uint64_t p = offs[i]; p < offs[i + 1]; ++p) {
      if (cols[p] < (uint64_t)i) {
        lci.push_back((int32_t)cols[p]);
        lv.push_back(lu[p]);
      } else {
        uci.push_back((int32_t)cols[p]);
        uv.push_back(lu[p]);
      }
    }
    lrp[i + 1] = (int64_t)lci.size();
    urp[i + 1] = (int64_t)uci.size();
  }
  std::vector<int32_t> lperm, uperm;
  std::vector<int64_t> llev, ulev;
  level_schedule(n, lrp, lci, true, lperm, llev);
  level_schedule(n, urp, uci, false, uperm, ulev);
  d.n = n;
  d.nnz_l = (int64_t)lv.size();
  d.nnz_u = (int64_t)uv.size();
  d.nlev_l = (int)llev.size() - 1;
  d.nlev_u = (int)ulev.size() - 1;
  // a 5-point grid (the base operator recognized the pattern): factors by neighbour
  if (d.base.d.kind == kStencilDia && d.base.d.dim == 2 && n <= 0x7fffffff) {
    const int64_t nx = d.base.d.nx;
    std::vector<double> lS(n, 0.0), lW(n, 0.0), uC(n, 0.0), uE(n, 0.0), uN(n, 0.0);
    std::vector<uint8_t> lm(n, 0), um(n, 0);
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i)
      for (uint64_t p = offs[i]; p < offs[i + 1]; ++p) {
        const int64_t off = (int64_t)cols[p] - i;
        if (off == -nx) lS[i] = lu[p], lm[i] |= 1;
        else if (off == -1) lW[i] = lu[p], lm[i] |= 2;
        else if (off == 0) uC[i] = lu[p];
        else if (off == 1) uE[i] = lu[p], um[i] |= 1;
        else if (off == nx) uN[i] = lu[p], um[i] |= 2;
        else ok = false;
      }
    if (ok) {
      d.gnx = nx;
      d.gny = d.base.d.ny;
      d.lS = upload(op, lS);
      d.lW = upload(op, lW);
      d.uC = upload(op, uC);
      d.uE = upload(op, uE);
      d.uN = upload(op, uN);
      d.lm = upload(op, lm);
      d.um = upload(op, um);
      std::vector<double> bnd((size_t)((nx + 31) / 32) * d.base.d.ny, 0.0);
      d.bnd = const_cast<double*>(upload(op, bnd));
      std::vector<int> st(1, 0);
      d.stalled = const_cast<int*>(upload(op, st));
    }
  }
  for (size_t q = 0; q + 1 < llev.size(); ++q) d.maxw_l = std::max(d.maxw_l, llev[q + 1] - llev[q]);
  for (size_t q = 0; q + 1 < ulev.size(); ++q) d.maxw_u = std::max(d.maxw_u, ulev[q + 1] - ulev[q]);
  d.lrp = upload(op, lrp);
  d.lci = upload(op, lci);
  d.lv = upload(op, lv);
  d.urp = upload(op, urp);
  d.uci = upload(op, uci);
  d.uv = upload(op, uv);
  d.lperm = upload(op, lperm);
  d.uperm = upload(op, uperm);
  d.llev = upload(op, llev);
  d.ulev = upload(op, ulev);
  op.device = c.device;
  op.n = n;
  op.rows = n;
  std::memset(&op.d, 0, sizeof op.d);
  op.d.kind = kIlu0;
  op.d.n = n;
  op.d.ilu = op.ilu.get();
}

// the strip solves' stall flag (a neighbour strip that never delivered its boundary column)
void ilu0_check(Ctx& c, const Op& op) {
  if (op.d.kind != kIlu0 || !op.ilu || !op.ilu->stalled) return;
  int h = 0;
  CK(cudaMemcpyAsync(&h, op.ilu->stalled, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (h) {
    const int z = 0;
    CK(cudaMemcpy(op.ilu->stalled, &z, sizeof z, cudaMemcpyHostToDevice));
    fail(SKC_ECUDA, "ilu0 strip solve: a neighbouring strip stalled past the spin limit");
  }
}

// z = (LU)^{-1} r (ilu0_apply); r may alias z
void launch_ilu0_solve(Ctx& c, const IluData& d, const double* r, double* z, const int* halt, const int* cond) {
  launch_trsv<true>(c, d, r, z, halt, cond);
  launch_trsv<false>(c, d, z, z, halt, cond);
  CK(cudaGetLastError());
}

}  // namespace skc
