// ref_caller.cpp -- caller code written against the reference's public API (namespace skrylov,
// SparseMatrix / as_operator / LinearOperator / SStepConfig / SolveReport / SStepBasis), in the
// shape of the reference's own call sites: a method dispatcher like detail::dispatch_method
// (bench.hpp:111-122) and the sarnoldi checks of test_sstep.cpp:276-311.  The only line that
// names this library is the include.  Prints one JSON object.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "skrylov_b200/skrylov.hpp"

using namespace skrylov;

namespace {

// 2D five-point convection-diffusion, natural ordering, h^2-scaled (the BASELINE operator)
SparseMatrix five_point(std::size_t nx, double conv) {
  const double h = 1.0 / (static_cast<double>(nx) + 1.0), ch2 = conv * h / 2.0;
  const std::size_t n = nx * nx;
  std::vector<std::size_t> offs{0}, cols;
  std::vector<double> vals;
  for (std::size_t j = 0; j < nx; ++j)
    for (std::size_t i = 0; i < nx; ++i) {
      const std::size_t p = j * nx + i;
      if (j > 0) cols.push_back(p - nx), vals.push_back(-1.0 - ch2);
      if (i > 0) cols.push_back(p - 1), vals.push_back(-1.0 - ch2);
      cols.push_back(p), vals.push_back(4.0);
      if (i + 1 < nx) cols.push_back(p + 1), vals.push_back(-1.0 + ch2);
      if (j + 1 < nx) cols.push_back(p + nx), vals.push_back(-1.0 + ch2);
      offs.push_back(cols.size());
    }
  return SparseMatrix(n, n, std::move(offs), std::move(cols), std::move(vals));
}

struct MethodSpec {
  std::string method;
  std::size_t s = 2, k = 2, m = 5;
};

SolveReport dispatch(const LinearOperator& op, std::span<const double> rhs, std::vector<double>& x,
                     const MethodSpec& ms, double threshold, std::size_t max_iterations) {
  SStepConfig cfg;
  cfg.s = ms.s;
  cfg.k = ms.k;
  cfg.m = ms.m;
  cfg.tol = threshold;
  cfg.max_iterations = max_iterations;
  cfg.unbounded_window = ms.method == "sgcr";
  if (ms.method == "smr") return smr_solve(op, rhs, x, cfg);
  if (ms.method == "somin" || ms.method == "sgcr") return somin_solve(op, rhs, x, cfg);
  if (ms.method == "sgmres") return sgmres_solve(op, rhs, x, cfg);
  throw std::invalid_argument("unknown method: " + ms.method);
}

double true_residual(const LinearOperator& op, std::span<const double> f, const std::vector<double>& x) {
  std::vector<double> ax = op(x);
  double acc = 0.0;
  for (std::size_t i = 0; i < f.size(); ++i) acc += (f[i] - ax[i]) * (f[i] - ax[i]);
  return std::sqrt(acc);
}

}  // namespace

int main(int argc, char** argv) {
  const std::size_t nx = argc > 1 ? std::stoul(argv[1]) : 48;
  SparseMatrix a = five_point(nx, 10.0);
  LinearOperator op = as_operator(a);
  LinearOperator copy = op;  // value semantics, like the reference's type-erased operator
  const std::size_t n = op.size();
  std::vector<double> f(n);
  for (std::size_t i = 0; i < n; ++i) f[i] = std::sin(0.37 * static_cast<double>(i) + 0.1);
  double fn = 0.0;
  for (double v : f) fn += v * v;
  const double tol = 1e-8 * std::sqrt(fn);

  std::printf("{\"n\": %zu, \"tol\": %.17g", n, tol);
  for (const char* m : {"somin", "sgcr", "sgmres", "smr"}) {
    MethodSpec ms;
    ms.method = m;
    ms.s = 2;
    std::vector<double> x(n, 0.0);
    const SolveReport rep = dispatch(copy, f, x, ms, tol, 100000);
    std::printf(", \"%s\": {\"converged\": %s, \"iterations\": %zu, \"history\": %zu, \"true_residual\": %.17g, "
                "\"final_residual\": %.17g, \"matvecs\": %llu}",
                m, rep.converged ? "true" : "false", rep.iterations, rep.residual_history.size(),
                true_residual(op, f, x), rep.final_residual, (unsigned long long)rep.op_counts.matvecs);
  }
  // smr_step with a caller-owned counter (sstep.hpp:89-107)
  {
    std::vector<double> x(n, 0.0), r = f;
    OpCounter c;
    std::vector<double> coef = smr_step(op, x, r, 3, &c);
    std::printf(", \"smr_step\": {\"coeffs\": %zu, \"matvecs\": %llu}", coef.size(), (unsigned long long)c.matvecs);
  }
  // sarnoldi: A V = U G with the returned blocks / hess / next seed (test_sstep.cpp:276-311)
  {
    const std::size_t s = 3, mb = 4;
    OpCounter c;
    SStepBasis b = sarnoldi(op, f, s, mb, &c);
    double err2 = 0.0, ref2 = 0.0;
    for (std::size_t bc = 0; bc < mb; ++bc)
      for (std::size_t lc = 0; lc < s; ++lc) {
        std::vector<double> av = op(b.blocks[bc].column(lc));
        const std::size_t col = bc * s + lc;
        for (std::size_t br = 0; br < mb; ++br)
          for (std::size_t lr = 0; lr < s; ++lr) {
            const double g = b.hess(br * s + lr, col);
            const auto v = b.blocks[br].column(lr);
            for (std::size_t i = 0; i < n; ++i) av[i] -= g * v[i];
          }
        const double g = b.hess(mb * s, col);
        for (std::size_t i = 0; i < n; ++i) av[i] -= g * b.next_seed[i];
        for (double v : av) err2 += v * v;
      }
    for (double v : a.values()) ref2 += v * v;
    std::printf(", \"sarnoldi\": {\"blocks\": %zu, \"width\": %zu, \"hess_rows\": %zu, \"hess_cols\": %zu, "
                "\"gram0_trace\": %.17g, \"avug_rel\": %.3e, \"dotprods\": %llu}",
                b.blocks.size(), b.blocks[0].width(), b.hess.rows(), b.hess.cols(), b.grams[0].trace(),
                std::sqrt(err2) / std::sqrt(ref2), (unsigned long long)c.dotprods);
  }
  // a host closure cannot run on the device: invalid_argument, no CPU fallback
  {
    LinearOperator host(n, [](std::span<const double> x, std::span<double> y) {
      for (std::size_t i = 0; i < x.size(); ++i) y[i] = x[i];
    });
    std::vector<double> x(n, 0.0);
    bool threw = false;
    try {
      SStepConfig cfg;
      somin_solve(host, f, x, cfg);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    bool bad_s = false;
    try {
      SStepConfig cfg;
      cfg.s = 9;
      somin_solve(op, f, x, cfg);
    } catch (const std::invalid_argument&) {
      bad_s = true;
    }
    std::printf(", \"host_closure_rejected\": %s, \"invalid_s_throws\": %s", threw ? "true" : "false",
                bad_s ? "true" : "false");
  }
  std::printf("}\n");
  return 0;
}
