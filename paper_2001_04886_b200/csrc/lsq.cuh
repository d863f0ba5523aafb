// lsq.cuh -- the least-squares half of s-step GMRES on the device (BASELINE north_star item 4):
// the incremental Givens QR of the block Hessenberg system (HessenbergLsq,
// small_dense.hpp:239-307), its back substitution with the rank check, and the glue of
// sgmres_solve's cycle loop -- the block Hessenberg column reconstruction (append_g_columns,
// sstep.hpp:422-445), the L scaling (apply_l, sstep.hpp:566-579) with the upper Cholesky factor
// of each basis block (cholesky_upper, small_dense.hpp:190-206) and the early exit rho <= tol
// (sstep.hpp:600).
//
// Layout: R is stored packed by columns (column j = rows 0..j at offset j(j+1)/2), the Givens
// pairs and the rotated right-hand side in flat arrays; everything lives in one workspace that
// persists across the kernels of a restart cycle.  The per-element arithmetic is the
// reference's (IEEE mul/add/div/sqrt without contraction, hypot via sd_hypot = the host C
// library's bits), so the residual estimates and y equal what the host computes from the same
// columns.  The serial primitives are SKC_HD: the C ABI's host hook skc_hessenberg_lsq runs the
// same code on the CPU.
#pragma once

#include <cstddef>
#include <cstdint>

#include "small_dense.cuh"

namespace skc {

struct LsqHdr {
  int cols;      // columns appended
  int rank_col;  // last back substitution: 1-based column of a rank-deficient diagonal, 0 = ok
  int pad0, pad1;
  double residual;  // |rhs[cols]|, the least-squares residual of the system so far
  double gnorm_sq;  // sum of squares of every appended (unrotated) entry, in append order
};

struct LsqView {
  int M;  // column capacity
  LsqHdr* h;
  double* cs;   // [M]
  double* sn;   // [M]
  double* rhs;  // [M + 1]
  double* R;    // packed columns, [M (M + 1) / 2]
  double* y;    // [M]
};

// doubles after the header for capacity M
SKC_HD size_t lsq_doubles(int M) { return (size_t)M * 4 + 1 + (size_t)M * (M + 1) / 2; }  // cs sn rhs R y
inline size_t lsq_bytes(int M) { return sizeof(LsqHdr) + lsq_doubles(M) * sizeof(double); }
SKC_HD LsqView lsq_view(void* base, int M) {
  LsqView v;
  v.M = M;
  v.h = reinterpret_cast<LsqHdr*>(base);
  double* p = reinterpret_cast<double*>(reinterpret_cast<char*>(base) + sizeof(LsqHdr));
  v.cs = p;
  v.sn = p + M;
  v.rhs = p + 2 * M;
  v.R = p + 3 * M + 1;
  v.y = v.R + (size_t)M * (M + 1) / 2;
  return v;
}
SKC_HD double& lsq_r(const LsqView& v, int col, int row) { return v.R[(size_t)col * (col + 1) / 2 + row]; }

// HessenbergLsq(beta) (small_dense.hpp:241)
SKC_HD void lsq_reset(const LsqView& v, double beta) {
  v.h->cols = 0;
  v.h->rank_col = 0;
  v.h->residual = sd_abs(beta);
  v.h->gnorm_sq = 0.0;
  v.rhs[0] = beta;
}

// one stored rotation applied to entries (t, t+1) of a column (small_dense.hpp:262-266)
SKC_HD void lsq_rotate(double c, double s, double* col, int t) {
  const double a = col[t], b = col[t + 1];
  col[t] = c * a + s * b;
  col[t + 1] = -s * a + c * b;
}

// The new rotation of column j (already rotated by 0..j-1) and the right-hand side update
// (small_dense.hpp:267-283); returns the new residual.
SKC_HD double lsq_finish_column(const LsqView& v, double* col, int j) {
  const double a = col[j], b = col[j + 1];
  const double r = sd_hypot(a, b);
  double c = 1.0, s = 0.0;
  if (r != 0.0) {
    c = a / r;
    s = b / r;
  }
  v.cs[j] = c;
  v.sn[j] = s;
  col[j] = r;
  for (int i = 0; i <= j; ++i) lsq_r(v, j, i) = col[i];
  v.rhs[j + 1] = 0.0;
  const double ra = v.rhs[j], rb = v.rhs[j + 1];
  v.rhs[j] = c * ra + s * rb;
  v.rhs[j + 1] = -s * ra + c * rb;
  v.h->residual = sd_abs(v.rhs[j + 1]);
  v.h->cols = j + 1;
  return v.h->residual;
}

// append_column, serial (small_dense.hpp:255-284): col has j + 2 entries, rotated in place
SKC_HD double lsq_append_serial(const LsqView& v, double* col) {
  const int j = v.h->cols;
  double g = v.h->gnorm_sq;
  for (int i = 0; i < j + 2; ++i) g += col[i] * col[i];
  v.h->gnorm_sq = g;
  for (int t = 0; t < j; ++t) lsq_rotate(v.cs[t], v.sn[t], col, t);
  return lsq_finish_column(v, col, j);
}

// solve() (small_dense.hpp:287-300): back substitution into v.y; false (rank_col set) when a
// diagonal of R is at or below 1e-14 ||G||_F -- unless `fixed` (fixed-step benchmark mode)
SKC_HD bool lsq_solve(const LsqView& v, bool fixed) {
  const int m = v.h->cols;
  const double tol = 1e-14 * sqrt(v.h->gnorm_sq);
  for (int i = 0; i < m; ++i) v.y[i] = 0.0;
  v.h->rank_col = 0;
  for (int ii = m - 1; ii >= 0; --ii) {
    double acc = v.rhs[ii];
    for (int k = ii + 1; k < m; ++k) acc -= lsq_r(v, k, ii) * v.y[k];
    if (sd_abs(lsq_r(v, ii, ii)) <= tol && !fixed) {
      v.h->rank_col = ii + 1;
      return false;
    }
    v.y[ii] = acc / lsq_r(v, ii, ii);
  }
  return true;
}

#ifdef __CUDACC__
// append_column for nc consecutive columns, whole CTA (>= 64 threads).  Column c lives at
// cols + c * ld with entries 0 .. j0 + c + 1 (j0 = columns already appended) and is rotated in
// place.  The squared norms accumulate on thread 0 in the reference's entry order from a copy
// (`copy`, nc * ld doubles) while warp 1 applies the stored rotations -- lane c to column c for
// the old pairs, then lane 0 the pairs created inside this batch, column by column.  res_out[c]
// (optional) = the residual after column c.  Ends with a barrier.
__device__ inline void lsq_append_cta(const LsqView& v, double* cols, int ld, int nc, double* copy, double* res_out) {
  __syncthreads();
  const int j0 = v.h->cols;
  for (int q = threadIdx.x; q < nc * ld; q += blockDim.x) {
    const int c = q / ld, r = q - c * ld;
    if (r < j0 + c + 2) copy[q] = cols[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = v.h->gnorm_sq;
    for (int c = 0; c < nc; ++c)
      for (int i = 0; i < j0 + c + 2; ++i) g += copy[c * ld + i] * copy[c * ld + i];
    v.h->gnorm_sq = g;
  } else if (threadIdx.x >= 32 && threadIdx.x < 64) {
    const int c = threadIdx.x - 32;
    if (c < nc) {
      double* col = cols + c * ld;
      for (int t = 0; t < j0; ++t) lsq_rotate(v.cs[t], v.sn[t], col, t);
    }
    __syncwarp();
    if (c == 0) {
      for (int cc = 0; cc < nc; ++cc) {
        double* col = cols + cc * ld;
        const int j = j0 + cc;
        for (int t = j0; t < j; ++t) lsq_rotate(v.cs[t], v.sn[t], col, t);
        const double res = lsq_finish_column(v, col, j);
        if (res_out) res_out[cc] = res;
      }
    }
  }
  __syncthreads();
}
#endif

}  // namespace skc
