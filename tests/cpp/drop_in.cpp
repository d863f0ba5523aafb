// Reference-style caller written against the drop-in header: the C1 operator as CSR, solved
// with s-step Orthomin and s-step GMRES exactly as a skrylov user would call the reference.
// Prints one JSON line; tests/test_cpp_dropin.py builds it (CPU) and runs it (GPU).
#include <cmath>
#include <cstdio>
#include <vector>

#include "skrylov_b200/sstep.hpp"

using namespace skrylov::b200;

int main(int argc, char** argv) {
  const std::size_t nx = argc > 1 ? std::stoul(argv[1]) : 64;
  const double conv = 10.0, h = 1.0 / (nx + 1.0), ch2 = conv * h / 2.0;
  const std::size_t n = nx * nx;
  std::vector<std::size_t> offs{0}, cols;
  std::vector<double> vals;
  for (std::size_t j = 0; j < nx; ++j)
    for (std::size_t i = 0; i < nx; ++i) {
      const std::size_t row = j * nx + i;
      if (j > 0) cols.push_back(row - nx), vals.push_back(-1.0 - ch2);
      if (i > 0) cols.push_back(row - 1), vals.push_back(-1.0 - ch2);
      cols.push_back(row), vals.push_back(4.0);
      if (i + 1 < nx) cols.push_back(row + 1), vals.push_back(-1.0 + ch2);
      if (j + 1 < nx) cols.push_back(row + nx), vals.push_back(-1.0 + ch2);
      offs.push_back(cols.size());
    }
  std::vector<double> f(n);
  for (std::size_t i = 0; i < n; ++i) f[i] = std::sin(0.37 * static_cast<double>(i));
  double fn = 0.0;
  for (double v : f) fn += v * v;
  fn = std::sqrt(fn);

  Context ctx(0);
  DeviceOperator op = ctx.csr(offs, cols, vals);
  SStepConfig cfg;
  cfg.s = 4;
  cfg.k = 2;
  cfg.tol = 1e-8 * fn;
  std::vector<double> x(n, 0.0);
  SolveReport a = somin_solve(op, f, x, cfg);
  auto ax = op(x);
  double tr = 0.0;
  for (std::size_t i = 0; i < n; ++i) tr += (f[i] - ax[i]) * (f[i] - ax[i]);
  cfg.s = 2;
  cfg.m = 5;
  std::vector<double> x2(n, 0.0);
  SolveReport b = sgmres_solve(op, f, x2, cfg);
  bool threw = false;
  try {
    cfg.s = 9;
    somin_solve(op, f, x2, cfg);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("{\"somin_converged\": %d, \"somin_iterations\": %zu, \"somin_true_residual\": %.17g, "
              "\"tol\": %.17g, \"sgmres_converged\": %d, \"sgmres_cycles\": %zu, \"invalid_s_throws\": %d}\n",
              a.converged, a.iterations, std::sqrt(tr), 1e-8 * fn, b.converged, b.cycles, threw);
  return 0;
}
