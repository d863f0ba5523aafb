// skrylov_b200/skrylov.hpp -- the reference's own namespace and types for the s-step path
// (/root/reference/proj/include/skrylov: sstep.hpp, operator.hpp, sparse.hpp, report.hpp,
// block.hpp, dense_matrix.hpp), backed by libskrylov_b200.so.  A reference caller switches by
// changing one include:
//     #include "skrylov/skrylov.hpp"   ->   #include "skrylov_b200/skrylov.hpp"
// and keeps its code: SparseMatrix, as_operator, LinearOperator, SStepConfig, SolveReport,
// OpCounter, SStepBasis (std::vector<DirectionBlock> blocks, std::vector<Matrix> grams, Matrix
// hess), breakdown_error and the solver calls somin_solve / sgmres_solve / smr_solve / smr_step /
// sarnoldi with the reference's signatures (sstep.hpp:89-91, 109-110, 142-143, 465-467,
// 493-494) and error behaviour.
//
// The one seam that changes is the operator: LinearOperator keeps the
// reference's value semantics and host apply(), and additionally carries a device-describable
// operator when it was made by as_operator(SparseMatrix) (pattern-detected 5/7-point grids run
// the stencil kernels) or stencil_operator(...).  A LinearOperator built from a host closure
// cannot run on the device: the solvers reject it with std::invalid_argument -- there is no CPU
// fallback.  Device work runs on a per-thread default context (device 0 unless
// set_default_device() chose another), as the reference's solves are call-confined and
// thread-compatible.
#ifndef SKRYLOV_B200_SKRYLOV_HPP
#define SKRYLOV_B200_SKRYLOV_HPP

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sstep.hpp"

namespace skrylov {

using breakdown_error = b200::breakdown_error;  // kernels.hpp:36-39

// kernels.hpp:41-43
inline void require(bool ok, const std::string& what) {
  if (!ok) throw std::invalid_argument(what);
}

// report.hpp:35-51
struct OpCounter {
  std::uint64_t dotprods = 0;
  std::uint64_t matvecs = 0;
  std::uint64_t vec_updates = 0;
  std::uint64_t stored_vectors = 0;
  std::uint64_t termination_dots = 0;
};
inline OpCounter operator-(const OpCounter& a, const OpCounter& b) {
  return {a.dotprods - b.dotprods, a.matvecs - b.matvecs, a.vec_updates - b.vec_updates,
          a.stored_vectors - b.stored_vectors, a.termination_dots - b.termination_dots};
}

// report.hpp:53-75 (+ block_rho: the per-block least-squares residuals of s-GMRES)
struct SolveReport {
  bool converged = false;
  std::size_t iterations = 0;
  std::size_t cycles = 0;
  std::vector<double> residual_history;
  double final_residual = 0.0;
  OpCounter op_counts;
  std::vector<OpCounter> op_history;
  std::size_t steady_iteration = 0;
  std::optional<std::string> breakdown;
  std::size_t fallback_cycles = 0;
  std::vector<std::string> notes;
  std::vector<double> block_rho;
};

// dense_matrix.hpp:32-80 (row-major)
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols, double fill = 0.0) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  double frobenius_norm() const {
    double acc = 0.0;
    for (double e : data_) acc += e * e;
    return std::sqrt(acc);
  }
  double trace() const {
    double acc = 0.0;
    for (std::size_t i = 0; i < rows_ && i < cols_; ++i) acc += (*this)(i, i);
    return acc;
  }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

// block.hpp:36-56: n x s, columns contiguous
class DirectionBlock {
 public:
  DirectionBlock() = default;
  DirectionBlock(std::size_t n, std::size_t s) : n_(n), s_(s), data_(n * s, 0.0) {
    require(s >= 1, "DirectionBlock: width must be at least 1");
  }
  std::size_t length() const { return n_; }
  std::size_t width() const { return s_; }
  std::span<double> column(std::size_t j) { return {data_.data() + j * n_, n_}; }
  std::span<const double> column(std::size_t j) const { return {data_.data() + j * n_, n_}; }

 private:
  std::size_t n_ = 0, s_ = 0;
  std::vector<double> data_;
};

namespace gpu {
// the calling thread's default device context (created on first use)
inline int& default_device() {
  thread_local int dev = 0;
  return dev;
}
inline b200::Context& context() {
  thread_local std::unique_ptr<b200::Context> ctx;
  thread_local int on = -1;
  if (!ctx || on != default_device()) {
    ctx = std::make_unique<b200::Context>(default_device());
    on = default_device();
  }
  return *ctx;
}
}  // namespace gpu
inline void set_default_device(int device) { gpu::default_device() = device; }

// operator.hpp:34-57, plus the device-describable operator (shared by copies)
class LinearOperator {
 public:
  using apply_fn = std::function<void(std::span<const double>, std::span<double>)>;

  LinearOperator() = default;
  LinearOperator(std::size_t n, apply_fn fn) : n_(n), fn_(std::move(fn)) {}
  explicit LinearOperator(std::shared_ptr<const b200::DeviceOperator> dev)
      : n_(dev->size()), dev_(std::move(dev)) {
    const b200::DeviceOperator* d = dev_.get();
    fn_ = [d](std::span<const double> x, std::span<double> y) { d->apply(x, y); };
  }

  std::size_t size() const { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const {
    require(x.size() == n_ && y.size() == n_, "LinearOperator: dimension mismatch");
    fn_(x, y);
  }
  std::vector<double> operator()(std::span<const double> x) const {
    std::vector<double> y(n_, 0.0);
    apply(x, y);
    return y;
  }
  // the device operator, or nullptr for a host closure
  const b200::DeviceOperator* device() const { return dev_.get(); }

 private:
  std::size_t n_ = 0;
  apply_fn fn_;
  std::shared_ptr<const b200::DeviceOperator> dev_;
};

// sparse.hpp:37-63 (size_t CSR, ascending columns per row, the reference's validation)
class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(std::size_t n_rows, std::size_t n_cols, std::vector<std::size_t> row_offsets,
               std::vector<std::size_t> col_indices, std::vector<double> values)
      : n_rows_(n_rows), n_cols_(n_cols), row_offsets_(std::move(row_offsets)), col_indices_(std::move(col_indices)),
        values_(std::move(values)) {
    require(row_offsets_.size() == n_rows_ + 1, "SparseMatrix: bad offset length");
    require(row_offsets_.front() == 0, "SparseMatrix: offsets must start at 0");
    require(row_offsets_.back() == values_.size() && col_indices_.size() == values_.size(),
            "SparseMatrix: offsets/values mismatch");
    for (std::size_t i = 0; i < n_rows_; ++i) {
      require(row_offsets_[i] <= row_offsets_[i + 1], "SparseMatrix: offsets must be non-decreasing");
      for (std::size_t p = row_offsets_[i]; p < row_offsets_[i + 1]; ++p) {
        require(col_indices_[p] < n_cols_, "SparseMatrix: column index out of range");
        require(p == row_offsets_[i] || col_indices_[p - 1] < col_indices_[p],
                "SparseMatrix: column indices must be strictly increasing within a row");
      }
    }
  }
  std::size_t rows() const { return n_rows_; }
  std::size_t cols() const { return n_cols_; }
  std::size_t nnz() const { return values_.size(); }
  std::span<const std::size_t> row_offsets() const { return row_offsets_; }
  std::span<const std::size_t> col_indices() const { return col_indices_; }
  std::span<const double> values() const { return values_; }

 private:
  std::size_t n_rows_ = 0, n_cols_ = 0;
  std::vector<std::size_t> row_offsets_, col_indices_;
  std::vector<double> values_;
};

// sparse.hpp:155-160: the matrix goes to the device (the operator owns its device copy, so
// unlike the reference the SparseMatrix need not outlive it)
inline LinearOperator as_operator(const SparseMatrix& a) {
  require(a.rows() == a.cols(), "as_operator: matrix must be square");
  auto dev = std::make_shared<b200::DeviceOperator>(gpu::context().csr(a.row_offsets(), a.col_indices(), a.values()));
  return LinearOperator(std::shared_ptr<const b200::DeviceOperator>(std::move(dev)));
}

// GPU addition: an h^2-scaled 5/7-point convection-diffusion stencil with coefficients
// generated on the fly (skrylov_b200.h skc_stencil_desc; kcell: per-cell k, n entries)
inline LinearOperator stencil_operator(const skc_stencil_desc& d, const double* kcell = nullptr) {
  auto dev = std::make_shared<b200::DeviceOperator>(gpu::context().stencil(d, kcell));
  return LinearOperator(std::shared_ptr<const b200::DeviceOperator>(std::move(dev)));
}

// sstep.hpp:48-58
struct SStepConfig {
  std::size_t s = 2;
  std::size_t k = 2;
  std::size_t m = 5;
  double tol = 1e-6;
  std::size_t max_iterations = 100000;
  bool precondition = false;
  bool unbounded_window = false;
  bool debug_checks = false;
  double divergence_factor = 10.0;
  bool fixed_steps = false;  // not in the reference: benchmark mode (skrylov_b200.h)
};

// sstep.hpp:256-262
struct SStepBasis {
  std::vector<DirectionBlock> blocks;
  std::vector<Matrix> grams;
  Matrix hess;
  std::vector<double> next_seed;
  double next_seed_norm = 0.0;
};

namespace detail {
inline const b200::DeviceOperator& device_of(const LinearOperator& op) {
  require(op.device() != nullptr,
          "skrylov_b200: the GPU solvers need a device-describable operator (as_operator(SparseMatrix) or "
          "stencil_operator); a host-closure LinearOperator cannot run on the device");
  return *op.device();
}
inline b200::SStepConfig to_b200(const SStepConfig& c) {
  b200::SStepConfig o;
  o.s = c.s;
  o.k = c.k;
  o.m = c.m;
  o.tol = c.tol;
  o.max_iterations = c.max_iterations;
  o.precondition = c.precondition;
  o.unbounded_window = c.unbounded_window;
  o.debug_checks = c.debug_checks;
  o.divergence_factor = c.divergence_factor;
  o.fixed_steps = c.fixed_steps;
  return o;
}
inline OpCounter from_b200(const b200::OpCounter& c) {
  return {c.dotprods, c.matvecs, c.vec_updates, c.stored_vectors, c.termination_dots};
}
inline SolveReport from_b200(b200::SolveReport&& r) {
  SolveReport o;
  o.converged = r.converged;
  o.iterations = r.iterations;
  o.cycles = r.cycles;
  o.residual_history = std::move(r.residual_history);
  o.final_residual = r.final_residual;
  o.op_counts = from_b200(r.op_counts);
  for (const auto& c : r.op_history) o.op_history.push_back(from_b200(c));
  o.steady_iteration = r.steady_iteration;
  o.breakdown = std::move(r.breakdown);
  o.fallback_cycles = r.fallback_cycles;
  o.notes = std::move(r.notes);
  o.block_rho = std::move(r.block_rho);
  return o;
}
}  // namespace detail

// sstep.hpp:142-143
inline SolveReport somin_solve(const LinearOperator& op, std::span<const double> f, std::vector<double>& x,
                               const SStepConfig& cfg) {
  return detail::from_b200(b200::somin_solve(detail::device_of(op), f, x, detail::to_b200(cfg)));
}
// sstep.hpp:493-494
inline SolveReport sgmres_solve(const LinearOperator& op, std::span<const double> f, std::vector<double>& x,
                                const SStepConfig& cfg) {
  return detail::from_b200(b200::sgmres_solve(detail::device_of(op), f, x, detail::to_b200(cfg)));
}
// sstep.hpp:109-110
inline SolveReport smr_solve(const LinearOperator& op, std::span<const double> f, std::vector<double>& x,
                             const SStepConfig& cfg) {
  return detail::from_b200(b200::smr_solve(detail::device_of(op), f, x, detail::to_b200(cfg)));
}
// sstep.hpp:89-91
inline std::vector<double> smr_step(const LinearOperator& op, std::vector<double>& x, std::vector<double>& r,
                                    std::size_t s, OpCounter* counter = nullptr) {
  require(s >= 1, "smr_step: s must be at least 1");
  b200::OpCounter c{};
  if (counter) c = {counter->dotprods, counter->matvecs, counter->vec_updates, counter->stored_vectors,
                    counter->termination_dots};
  std::vector<double> a = b200::smr_step(detail::device_of(op), x, r, s, &c);
  if (counter) *counter = detail::from_b200(c);
  return a;
}
// sstep.hpp:465-485
inline SStepBasis sarnoldi(const LinearOperator& op, std::span<const double> v1, std::size_t s, std::size_t m_blocks,
                           OpCounter* counter = nullptr) {
  b200::OpCounter c{};
  if (counter) c = {counter->dotprods, counter->matvecs, counter->vec_updates, counter->stored_vectors,
                    counter->termination_dots};
  const b200::SStepBasis flat = b200::sarnoldi(detail::device_of(op), v1, s, m_blocks, &c);
  if (counter) *counter = detail::from_b200(c);
  const std::size_t n = op.size();
  SStepBasis b;
  for (std::size_t i = 0; i < m_blocks; ++i) {
    DirectionBlock blk(n, s);
    for (std::size_t j = 0; j < s; ++j) {
      const double* src = flat.blocks.data() + (i * s + j) * n;
      std::copy(src, src + n, blk.column(j).begin());
    }
    b.blocks.push_back(std::move(blk));
    Matrix g(s, s);
    for (std::size_t r = 0; r < s; ++r)
      for (std::size_t q = 0; q < s; ++q) g(r, q) = flat.grams[i * s * s + r * s + q];
    b.grams.push_back(std::move(g));
  }
  const std::size_t rows = (m_blocks + 1) * s, cols = m_blocks * s;
  b.hess = Matrix(rows, cols);
  for (std::size_t r = 0; r < rows; ++r)
    for (std::size_t q = 0; q < cols; ++q) b.hess(r, q) = flat.hess[r * cols + q];
  b.next_seed = flat.next_seed;
  b.next_seed_norm = flat.next_seed_norm;
  return b;
}

}  // namespace skrylov

#endif  // SKRYLOV_B200_SKRYLOV_HPP
