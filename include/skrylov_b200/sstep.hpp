// skrylov_b200/sstep.hpp -- header-only C++20 drop-in for the reference solver API
// (/root/reference/proj/include/skrylov/sstep.hpp), backed by libskrylov_b200.so through the
// C ABI in skrylov_b200.h.
//
// A reference caller switches by replacing
//     #include "skrylov/sstep.hpp"          ->  #include "skrylov_b200/sstep.hpp"
//     using namespace skrylov;              ->  using namespace skrylov::b200;
//     LinearOperator op = as_operator(a);   ->  DeviceOperator op = ctx.csr(a_offsets, a_cols, a_vals);
// The solver calls (somin_solve, sgmres_solve, smr_solve, smr_step, sarnoldi), SStepConfig,
// SolveReport and OpCounter keep the reference's names, fields, argument meaning and error
// behaviour (std::invalid_argument for require(), breakdown_error, std::logic_error).
#ifndef SKRYLOV_B200_SSTEP_HPP
#define SKRYLOV_B200_SSTEP_HPP

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../skrylov_b200.h"

namespace skrylov::b200 {

class breakdown_error : public std::runtime_error {  // kernels.hpp:36-39
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == SKC_OK) return;
  const std::string msg = skc_last_error();
  switch (status) {
    case SKC_EINVAL: throw std::invalid_argument(msg);
    case SKC_EBREAKDOWN: throw breakdown_error(msg);
    case SKC_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

using OpCounter = skc_op_counter;  // report.hpp:35-41 (same fields)

struct SStepConfig {  // sstep.hpp:48-58 (same defaults)
  std::size_t s = 2;
  std::size_t k = 2;
  std::size_t m = 5;
  double tol = 1e-6;
  std::size_t max_iterations = 100000;
  bool precondition = false;
  bool unbounded_window = false;
  bool debug_checks = false;
  double divergence_factor = 10.0;
  bool fixed_steps = false;  // not in the reference: benchmark mode (see skrylov_b200.h)

  skc_sstep_config c() const {
    return {s, k, m, tol, max_iterations, precondition, unbounded_window, debug_checks, divergence_factor,
            fixed_steps};
  }
};

struct SolveReport {  // report.hpp:53-75 (+ block_rho)
  bool converged = false;
  std::size_t iterations = 0;
  std::size_t cycles = 0;
  std::vector<double> residual_history;
  double final_residual = 0.0;
  OpCounter op_counts{};
  std::vector<OpCounter> op_history;
  std::size_t steady_iteration = 0;
  std::optional<std::string> breakdown;
  std::size_t fallback_cycles = 0;
  std::vector<std::string> notes;
  std::vector<double> block_rho;
};

namespace detail {
class Report {
 public:
  Report() { check(skc_report_create(&h_)); }
  ~Report() { skc_report_destroy(h_); }
  Report(const Report&) = delete;
  Report& operator=(const Report&) = delete;
  skc_report* get() { return h_; }
  SolveReport collect() const {
    skc_report_summary s{};
    check(skc_report_get_summary(h_, &s));
    SolveReport r;
    r.converged = s.converged;
    r.iterations = s.iterations;
    r.cycles = s.cycles;
    r.final_residual = s.final_residual;
    r.op_counts = s.op_counts;
    r.steady_iteration = s.steady_iteration;
    r.fallback_cycles = s.fallback_cycles;
    r.residual_history.resize(s.n_history);
    skc_report_get_history(h_, r.residual_history.data(), s.n_history);
    r.op_history.resize(s.n_op_history);
    skc_report_get_op_history(h_, r.op_history.data(), s.n_op_history);
    r.block_rho.resize(s.n_block_rho);
    skc_report_get_block_rho(h_, r.block_rho.data(), s.n_block_rho);
    if (s.has_breakdown) {
      std::string b(skc_report_get_breakdown(h_, nullptr, 0), '\0');
      skc_report_get_breakdown(h_, b.data(), b.size() + 1);
      r.breakdown = b;
    }
    for (uint64_t i = 0; i < s.n_notes; ++i) {
      std::string nt(skc_report_get_note(h_, i, nullptr, 0), '\0');
      skc_report_get_note(h_, i, nt.data(), nt.size() + 1);
      r.notes.push_back(nt);
    }
    return r;
  }

 private:
  skc_report* h_ = nullptr;
};
}  // namespace detail

class Context;

// Device-describable operator: the GPU counterpart of LinearOperator (operator.hpp:34-57).
class DeviceOperator {
 public:
  DeviceOperator(skc_ctx* ctx, skc_op* op) : ctx_(ctx), op_(op) { check(skc_op_size(op_, &n_)); }
  ~DeviceOperator() {
    if (op_) skc_op_destroy(op_);
  }
  DeviceOperator(DeviceOperator&& o) noexcept : ctx_(o.ctx_), op_(std::exchange(o.op_, nullptr)), n_(o.n_) {}
  DeviceOperator(const DeviceOperator&) = delete;
  DeviceOperator& operator=(const DeviceOperator&) = delete;

  std::size_t size() const { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const {
    if (x.size() != n_ || y.size() != n_) throw std::invalid_argument("LinearOperator: dimension mismatch");
    check(skc_op_apply(ctx_, op_, x.data(), y.data()));
  }
  std::vector<double> operator()(std::span<const double> x) const {
    std::vector<double> y(n_, 0.0);
    apply(x, y);
    return y;
  }
  skc_ctx* ctx() const { return ctx_; }
  skc_op* handle() const { return op_; }
  // z = (LU)^{-1} r for an operator made by Context::ilu0 (ilu0_apply, ilu0.hpp:99-134)
  std::vector<double> ilu0_apply(std::span<const double> r) const {
    if (r.size() != n_) throw std::invalid_argument("ilu0_apply: dimension mismatch");
    std::vector<double> z(n_, 0.0);
    check(skc_ilu0_solve(ctx_, op_, r.data(), z.data()));
    return z;
  }

 private:
  skc_ctx* ctx_;
  skc_op* op_;
  uint64_t n_ = 0;
};

// One context (device, stream, workspaces) per calling thread.
class Context {
 public:
  explicit Context(int device = 0) { check(skc_ctx_create(device, &h_)); }
  ~Context() { skc_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  skc_ctx* get() const { return h_; }

  // as_operator(SparseMatrix) (sparse.hpp:155-160)
  DeviceOperator csr(std::span<const std::size_t> row_offsets, std::span<const std::size_t> col_indices,
                     std::span<const double> values) const {
    static_assert(sizeof(std::size_t) == sizeof(uint64_t));
    skc_op* op = nullptr;
    check(skc_op_create_csr(h_, row_offsets.size() - 1, reinterpret_cast<const uint64_t*>(row_offsets.data()),
                            reinterpret_cast<const uint64_t*>(col_indices.data()), values.data(), &op));
    return DeviceOperator(h_, op);
  }
  DeviceOperator stencil(const skc_stencil_desc& d, const double* kcell = nullptr) const {
    skc_op* op = nullptr;
    check(skc_op_create_stencil(h_, &d, kcell, &op));
    return DeviceOperator(h_, op);
  }
  // right_preconditioned(a, ilu0_factor(a)) (ilu0.hpp:138-146, 45-95): A (LU)^{-1}; throws
  // breakdown_error "ilu0: zero pivot at row N" like ilu0_factor
  DeviceOperator ilu0(std::span<const std::size_t> row_offsets, std::span<const std::size_t> col_indices,
                      std::span<const double> values) const {
    skc_op* op = nullptr;
    check(skc_op_create_ilu0(h_, row_offsets.size() - 1, reinterpret_cast<const uint64_t*>(row_offsets.data()),
                             reinterpret_cast<const uint64_t*>(col_indices.data()), values.data(), &op));
    return DeviceOperator(h_, op);
  }

 private:
  skc_ctx* h_ = nullptr;
};

namespace detail {
template <class Fn>
SolveReport solve(Fn fn, const DeviceOperator& op, std::span<const double> f, std::vector<double>& x,
                  const SStepConfig& cfg) {
  if (f.size() != op.size() || x.size() != op.size())
    throw std::invalid_argument("solve: rhs/guess dimension mismatch");
  Report rep;
  const skc_sstep_config c = cfg.c();
  check(fn(op.ctx(), op.handle(), f.data(), x.data(), &c, rep.get()));
  return rep.collect();
}
}  // namespace detail

// sstep.hpp:142-143
inline SolveReport somin_solve(const DeviceOperator& op, std::span<const double> f, std::vector<double>& x,
                               const SStepConfig& cfg) {
  return detail::solve(skc_somin_solve, op, f, x, cfg);
}
// sstep.hpp:493-494
inline SolveReport sgmres_solve(const DeviceOperator& op, std::span<const double> f, std::vector<double>& x,
                                const SStepConfig& cfg) {
  return detail::solve(skc_sgmres_solve, op, f, x, cfg);
}
// sstep.hpp:109-110
inline SolveReport smr_solve(const DeviceOperator& op, std::span<const double> f, std::vector<double>& x,
                             const SStepConfig& cfg) {
  return detail::solve(skc_smr_solve, op, f, x, cfg);
}
// sstep.hpp:89-91
inline std::vector<double> smr_step(const DeviceOperator& op, std::vector<double>& x, std::vector<double>& r,
                                    std::size_t s, OpCounter* counter = nullptr) {
  std::vector<double> a(s, 0.0);
  OpCounter local{};
  check(skc_smr_step(op.ctx(), op.handle(), x.data(), r.data(), s, a.data(), counter ? counter : &local));
  return a;
}

struct SStepBasis {  // sstep.hpp:256-262 (blocks flattened: block b, column j at (b*s + j)*n)
  std::vector<double> blocks, grams, hess, next_seed;
  double next_seed_norm = 0.0;
};
// sstep.hpp:465-467
inline SStepBasis sarnoldi(const DeviceOperator& op, std::span<const double> v1, std::size_t s,
                           std::size_t m_blocks, OpCounter* counter = nullptr) {
  if (s < 1) throw std::invalid_argument("sarnoldi: s must be at least 1");
  if (m_blocks < 1) throw std::invalid_argument("sarnoldi: m_blocks must be at least 1");
  const std::size_t n = op.size();
  SStepBasis b;
  b.blocks.assign(m_blocks * s * n, 0.0);
  b.grams.assign(m_blocks * s * s, 0.0);
  b.hess.assign((m_blocks + 1) * s * m_blocks * s, 0.0);
  b.next_seed.assign(n, 0.0);
  check(skc_sarnoldi(op.ctx(), op.handle(), v1.data(), s, m_blocks, b.blocks.data(), b.grams.data(), b.hess.data(),
                     b.next_seed.data(), &b.next_seed_norm, counter));
  return b;
}

}  // namespace skrylov::b200

#endif  // SKRYLOV_B200_SSTEP_HPP
