// small_dense.cuh -- s x s Gram solves and the upper Cholesky factor, usable on the host
// and inside the single-CTA scalar kernels.
//
// Semantics follow GramSolver (small_dense.hpp:42-186) and cholesky_upper
// (small_dense.hpp:190-206): Cholesky with a 1e-13*|trace|/s pivot floor, falling back
// to LDL^T with symmetric diagonal pivoting; breakdown when min/max |pivot| < 1e-15.
// Every operation is an IEEE double add/sub/mul/div/sqrt in the reference's order and
// this file is compiled without FMA contraction (--fmad=false / -ffp-contract=off), so
// host and device produce the reference's bits for the same input matrix.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define SKC_HD __host__ __device__ __forceinline__
#else
#define SKC_HD inline
#endif

namespace skc {

constexpr int kMaxS = 8;  // validate_block_size: 1 <= s <= 8 (sstep.hpp:62-67)

// Gram factorization state; `ok` false means breakdown (the reference throws).
struct Gram {
  int order;
  int used_ldlt;
  int ok;
  int singular1;        // 1x1 zero system ("sym_solve: singular 1x1 Gram system")
  double ratio;         // min/max |pivot| (0 when all pivots vanish)
  double w[kMaxS * kMaxS];
  double fac[kMaxS * kMaxS];
  double piv[kMaxS];
  int perm[kMaxS];
};

SKC_HD double sd_abs(double v) { return v < 0.0 ? -v : v; }

SKC_HD double sd_trace(const double* w, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += w[i * n + i];
  return acc;
}

SKC_HD bool gram_try_cholesky(Gram& g) {
  const int n = g.order;
  const double floor_ = 1e-13 * sd_abs(sd_trace(g.w, n)) / static_cast<double>(n);
  for (int i = 0; i < n * n; ++i) g.fac[i] = 0.0;
  for (int i = 0; i < n; ++i) g.piv[i] = 0.0;
  for (int j = 0; j < n; ++j) {
    double d = g.w[j * n + j];
    for (int k = 0; k < j; ++k) d -= g.fac[j * n + k] * g.fac[j * n + k];
    if (d <= floor_) return false;
    g.piv[j] = d;
    g.fac[j * n + j] = sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double acc = g.w[i * n + j];
      for (int k = 0; k < j; ++k) acc -= g.fac[i * n + k] * g.fac[j * n + k];
      g.fac[i * n + j] = acc / g.fac[j * n + j];
    }
  }
  return true;
}

SKC_HD void gram_factor_ldlt(Gram& g) {
  const int n = g.order;
  double m[kMaxS * kMaxS];
  g.used_ldlt = 1;
  for (int i = 0; i < n * n; ++i) {
    m[i] = g.w[i];
    g.fac[i] = 0.0;
  }
  for (int i = 0; i < n; ++i) {
    g.perm[i] = i;
    g.piv[i] = 0.0;
  }
  for (int j = 0; j < n; ++j) {
    int p = j;
    for (int i = j + 1; i < n; ++i)
      if (sd_abs(m[i * n + i]) > sd_abs(m[p * n + p])) p = i;
    if (p != j) {
      for (int t = 0; t < n; ++t) {
        const double a = m[j * n + t];
        m[j * n + t] = m[p * n + t];
        m[p * n + t] = a;
      }
      for (int t = 0; t < n; ++t) {
        const double a = m[t * n + j];
        m[t * n + j] = m[t * n + p];
        m[t * n + p] = a;
      }
      for (int t = 0; t < j; ++t) {
        const double a = g.fac[j * n + t];
        g.fac[j * n + t] = g.fac[p * n + t];
        g.fac[p * n + t] = a;
      }
      const int q = g.perm[j];
      g.perm[j] = g.perm[p];
      g.perm[p] = q;
    }
    const double d = m[j * n + j];
    g.piv[j] = d;
    g.fac[j * n + j] = 1.0;
    if (d == 0.0) continue;
    for (int i = j + 1; i < n; ++i) g.fac[i * n + j] = m[i * n + j] / d;
    for (int i = j + 1; i < n; ++i)
      for (int k = j + 1; k <= i; ++k) {
        m[i * n + k] -= g.fac[i * n + j] * d * g.fac[k * n + j];
        m[k * n + i] = m[i * n + k];
      }
  }
}

// Factor W (row-major, order n). Sets g.ok / g.ratio / g.singular1.
SKC_HD void gram_factor(Gram& g, const double* w, int n) {
  g.order = n;
  g.used_ldlt = 0;
  g.ok = 1;
  g.singular1 = 0;
  g.ratio = 1.0;
  for (int i = 0; i < n * n; ++i) g.w[i] = w[i];
  if (n == 1) {
    g.piv[0] = w[0];
    if (w[0] == 0.0) {
      g.ok = 0;
      g.singular1 = 1;
      g.ratio = 0.0;
    }
    return;
  }
  if (!gram_try_cholesky(g)) gram_factor_ldlt(g);
  double pmin = sd_abs(g.piv[0]), pmax = pmin;
  for (int i = 0; i < n; ++i) {
    const double a = sd_abs(g.piv[i]);
    pmin = a < pmin ? a : pmin;
    pmax = a > pmax ? a : pmax;
  }
  g.ratio = pmax == 0.0 ? 0.0 : pmin / pmax;
  if (pmax == 0.0 || pmin / pmax < 1e-15) g.ok = 0;
}

// Fixed-step benchmark mode: accept a factorization the pivot-ratio test rejected
// (small_dense.hpp:62-64 is the only check skipped; a singular 1x1 system still fails)
SKC_HD void gram_bypass_ratio(Gram& g, int fixed) {
  if (fixed && !g.singular1) g.ok = 1;
}

// x = W^{-1} rhs (small_dense.hpp:75-112)
SKC_HD void gram_solve(const Gram& g, const double* rhs, double* x) {
  const int n = g.order;
  if (n == 1) {
    x[0] = rhs[0] / g.w[0];
    return;
  }
  if (!g.used_ldlt) {
    for (int i = 0; i < n; ++i) {
      double acc = rhs[i];
      for (int k = 0; k < i; ++k) acc -= g.fac[i * n + k] * x[k];
      x[i] = acc / g.fac[i * n + i];
    }
    for (int ii = n - 1; ii >= 0; --ii) {
      double acc = x[ii];
      for (int k = ii + 1; k < n; ++k) acc -= g.fac[k * n + ii] * x[k];
      x[ii] = acc / g.fac[ii * n + ii];
    }
    return;
  }
  double b[kMaxS];
  for (int i = 0; i < n; ++i) b[i] = rhs[g.perm[i]];
  for (int i = 0; i < n; ++i) {
    double acc = b[i];
    for (int k = 0; k < i; ++k) acc -= g.fac[i * n + k] * b[k];
    b[i] = acc;
  }
  for (int i = 0; i < n; ++i) b[i] /= g.piv[i];
  for (int ii = n - 1; ii >= 0; --ii) {
    double acc = b[ii];
    for (int k = ii + 1; k < n; ++k) acc -= g.fac[k * n + ii] * b[k];
    b[ii] = acc;
  }
  for (int i = 0; i < n; ++i) x[g.perm[i]] = b[i];
}

#ifdef __CUDACC__
// Compile-time-order versions for the device kernels: the same operations in the same order
// (hence the same bits) with every array in registers instead of local memory.  The LDL^T
// fallback (a failed Cholesky attempt: rare, ill-conditioned Gram matrices) takes the generic
// path above.
// the Cholesky path of gram_solve on the factor alone (row-major L, order N)
template <int N>
__device__ __forceinline__ void chol_solve_t(const double* fac, const double* rhs, double* x) {
  double f[N * N];
#pragma unroll
  for (int q = 0; q < N * N; ++q) f[q] = fac[q];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double acc = rhs[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc -= f[i * N + k] * x[k];
    x[i] = acc / f[i * N + i];
  }
#pragma unroll
  for (int ii = N - 1; ii >= 0; --ii) {
    double acc = x[ii];
#pragma unroll
    for (int k = ii + 1; k < N; ++k) acc -= f[k * N + ii] * x[k];
    x[ii] = acc / f[ii * N + ii];
  }
}

template <int N>
__device__ __forceinline__ void gram_solve_t(const Gram& g, const double* rhs, double* x) {
  if (N == 1 || g.used_ldlt) {
    // (the generic path through copies: the caller's arrays never have their address taken, so
    // they stay in registers on the common Cholesky path)
    double r2[kMaxS], x2[kMaxS];
#pragma unroll
    for (int i = 0; i < N; ++i) r2[i] = rhs[i];
    gram_solve(g, r2, x2);
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = x2[i];
    return;
  }
  chol_solve_t<N>(g.fac, rhs, x);
}

template <int N>
__device__ __forceinline__ void gram_factor_t(Gram& g, const double* w) {
  if (N == 1) {
    gram_factor(g, w, N);
    return;
  }
  g.order = N;
  g.used_ldlt = 0;
  g.ok = 1;
  g.singular1 = 0;
  double wr[N * N];
#pragma unroll
  for (int q = 0; q < N * N; ++q) g.w[q] = wr[q] = w[q];
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) tr += wr[i * N + i];
  const double floor_ = 1e-13 * sd_abs(tr) / static_cast<double>(N);
  double f[N * N], pv[N];
#pragma unroll
  for (int q = 0; q < N * N; ++q) f[q] = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) pv[i] = 0.0;
  bool chol = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if (chol) {
      double d = wr[j * N + j];
#pragma unroll
      for (int k = 0; k < j; ++k) d -= f[j * N + k] * f[j * N + k];
      if (d <= floor_) {
        chol = false;
      } else {
        pv[j] = d;
        f[j * N + j] = sqrt(d);
#pragma unroll
        for (int i = j + 1; i < N; ++i) {
          double acc = wr[i * N + j];
#pragma unroll
          for (int k = 0; k < j; ++k) acc -= f[i * N + k] * f[j * N + k];
          f[i * N + j] = acc / f[j * N + j];
        }
      }
    }
  }
  if (chol) {
#pragma unroll
    for (int q = 0; q < N * N; ++q) g.fac[q] = f[q];
#pragma unroll
    for (int i = 0; i < N; ++i) g.piv[i] = pv[i];
  } else {
    gram_factor_ldlt(g);
#pragma unroll
    for (int i = 0; i < N; ++i) pv[i] = g.piv[i];
  }
  double pmin = sd_abs(pv[0]), pmax = pmin;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double a = sd_abs(pv[i]);
    pmin = a < pmin ? a : pmin;
    pmax = a > pmax ? a : pmax;
  }
  g.ratio = pmax == 0.0 ? 0.0 : pmin / pmax;
  if (pmax == 0.0 || pmin / pmax < 1e-15) g.ok = 0;
}

// runtime order -> compile-time-order versions (device kernels whose order is a run-time
// argument)
__device__ __forceinline__ void gram_factor_dev(Gram& g, const double* w, int n) {
  switch (n) {
    case 2: gram_factor_t<2>(g, w); return;
    case 3: gram_factor_t<3>(g, w); return;
    case 4: gram_factor_t<4>(g, w); return;
    case 5: gram_factor_t<5>(g, w); return;
    case 6: gram_factor_t<6>(g, w); return;
    case 7: gram_factor_t<7>(g, w); return;
    case 8: gram_factor_t<8>(g, w); return;
    default: gram_factor(g, w, n);
  }
}
__device__ __forceinline__ void gram_solve_dev(const Gram& g, const double* rhs, double* x) {
  switch (g.order) {
    case 2: gram_solve_t<2>(g, rhs, x); return;
    case 3: gram_solve_t<3>(g, rhs, x); return;
    case 4: gram_solve_t<4>(g, rhs, x); return;
    case 5: gram_solve_t<5>(g, rhs, x); return;
    case 6: gram_solve_t<6>(g, rhs, x); return;
    case 7: gram_solve_t<7>(g, rhs, x); return;
    case 8: gram_solve_t<8>(g, rhs, x); return;
    default: gram_solve(g, rhs, x);
  }
}
#endif

// hypot(a, b) with the host C library's bits (glibc >= 2.35): the correction step of
// C. F. Borges, "An improved algorithm for hypot(a,b)" (2019) on the unfused path, with the
// power-of-two rescaling for huge / tiny operands.  Verified bit-identical to glibc 2.39's
// hypot on 2e7 random operand pairs spanning 40 decades.
// Compiled without contraction like the rest of this file.
SKC_HD double sd_hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
SKC_HD double sd_hypot(double x, double y) {
  x = sd_abs(x);
  y = sd_abs(y);
  if (isinf(x) || isinf(y)) return isinf(x) ? x : y;  // (an infinite operand wins over nan)
  if (isnan(x) || isnan(y)) return x + y;
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return sd_hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return sd_hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return sd_hypot_kernel(ax, ay);
}

// R^T R = W, upper triangular (small_dense.hpp:190-206). Returns false on breakdown.
SKC_HD bool cholesky_upper(const double* w, int n, double* r) {
  for (int i = 0; i < n * n; ++i) r[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    double d = w[i * n + i];
    for (int k = 0; k < i; ++k) d -= r[k * n + i] * r[k * n + i];
    if (d <= 0.0) return false;
    r[i * n + i] = sqrt(d);
    for (int j = i + 1; j < n; ++j) {
      double acc = w[i * n + j];
      for (int k = 0; k < i; ++k) acc -= r[k * n + i] * r[k * n + j];
      r[i * n + j] = acc / r[i * n + i];
    }
  }
  return true;
}

}  // namespace skc
