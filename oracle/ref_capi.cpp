// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the *unmodified* reference implementation (compiled from the headers
// under /root/reference/proj/include) through the same C ABI as the oracle
// restatement (skrylov_oracle.h, prefix ref_ instead of orc_).  Built by
// oracle/Makefile into oracle/_ref/libskref.so; used to pin the restatement and
// as the reference CPU arm of bench.py.  No reference source is copied here:
// this file only converts between C arrays and the reference's own types.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <random>

#include "skrylov/accounting.hpp"
#include "skrylov/ilu0.hpp"
#include "skrylov/kernels.hpp"
#include "skrylov/problem.hpp"
#include "skrylov/sparse.hpp"
#include "skrylov/sstep.hpp"
#include "skrylov/solvers.hpp"
#include "skrylov_oracle.h"

using namespace skrylov;

namespace {

SparseMatrix to_sparse(const orc_csr* a) {
  const std::size_t n = a->n;
  std::vector<std::size_t> offs(a->row_offsets, a->row_offsets + n + 1);
  const std::size_t nnz = offs.back();
  std::vector<std::size_t> cols(a->col_indices, a->col_indices + nnz);
  std::vector<double> vals(a->values, a->values + nnz);
  return SparseMatrix(n, n, std::move(offs), std::move(cols), std::move(vals));
}

orc_counter conv(const OpCounter& c) {
  return {c.dotprods, c.matvecs, c.vec_updates, c.stored_vectors, c.termination_dots};
}

void fill(orc_report* out, const SolveReport& rep) {
  out->converged = rep.converged;
  out->iterations = rep.iterations;
  out->cycles = rep.cycles;
  out->n_history = rep.residual_history.size();
  out->history = static_cast<double*>(std::malloc(sizeof(double) * (out->n_history + 1)));
  for (std::size_t i = 0; i < out->n_history; ++i) out->history[i] = rep.residual_history[i];
  out->final_residual = rep.final_residual;
  out->op_counts = conv(rep.op_counts);
  out->n_op_history = rep.op_history.size();
  out->op_history =
      static_cast<orc_counter*>(std::malloc(sizeof(orc_counter) * (out->n_op_history + 1)));
  for (std::size_t i = 0; i < out->n_op_history; ++i) out->op_history[i] = conv(rep.op_history[i]);
  out->steady_iteration = rep.steady_iteration;
  out->has_breakdown = rep.breakdown.has_value();
  if (rep.breakdown)
    std::snprintf(out->breakdown, sizeof out->breakdown, "%s", rep.breakdown->c_str());
  out->fallback_cycles = rep.fallback_cycles;
  out->n_notes = 0;
  for (const auto& s : rep.notes)
    if (out->n_notes < 4) std::snprintf(out->notes[out->n_notes++], 256, "%s", s.c_str());
}

SStepConfig sconf(const orc_sstep_cfg* c) {
  SStepConfig s;
  s.s = c->s;
  s.k = c->k;
  s.m = c->m;
  s.tol = c->tol;
  s.max_iterations = c->max_iterations;
  s.precondition = c->precondition;
  s.unbounded_window = c->unbounded_window;
  s.debug_checks = c->debug_checks;
  s.divergence_factor = c->divergence_factor;
  return s;
}

SolverConfig oconf(const orc_solver_cfg* c) {
  SolverConfig s;
  s.method = static_cast<Method>(c->method);
  s.k = c->k;
  s.m = c->m;
  s.tol = c->tol;
  s.max_iterations = c->max_iterations;
  s.precondition = c->precondition;
  s.debug_checks = c->debug_checks;
  s.divergence_factor = c->divergence_factor;
  return s;
}

template <class F>
int guarded(char* err, std::size_t cap, F&& body) {
  try {
    body();
    return 0;
  } catch (const breakdown_error& e) {
    if (err) std::snprintf(err, cap, "%s", e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    if (err) std::snprintf(err, cap, "%s", e.what());
    return 1;
  } catch (const std::logic_error& e) {
    if (err) std::snprintf(err, cap, "%s", e.what());
    return 3;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, cap, "%s", e.what());
    return 4;
  }
}

template <class Solve>
int run_solver(const orc_csr* a, const double* f, double* x, orc_report* rep, Solve&& solve) {
  return guarded(rep->error, sizeof rep->error, [&] {
    SparseMatrix m = to_sparse(a);
    LinearOperator op = as_operator(m);
    std::span<const double> fs(f, a->n);
    std::vector<double> xv(x, x + a->n);
    SolveReport r = solve(op, fs, xv);
    std::memcpy(x, xv.data(), sizeof(double) * a->n);
    fill(rep, r);
  });
}

}  // namespace

extern "C" {

void ref_report_init(orc_report* r) { std::memset(r, 0, sizeof *r); }
void ref_report_free(orc_report* r) {
  std::free(r->history);
  std::free(r->op_history);
  std::free(r->block_rho);
  std::memset(r, 0, sizeof *r);
}

void ref_spmv(const orc_csr* a, const double* x, double* y) {
  SparseMatrix m = to_sparse(a);
  spmv(m, std::span<const double>(x, a->n), std::span<double>(y, a->n));
}

int ref_krylov_block(const orc_csr* a, const double* v, uint64_t s, double* out) {
  return guarded(nullptr, 0, [&] {
    SparseMatrix m = to_sparse(a);
    LinearOperator op = as_operator(m);
    DirectionBlock b = krylov_block(op, std::span<const double>(v, a->n), s);
    for (std::size_t j = 0; j < s; ++j)
      std::memcpy(out + j * a->n, b.column(j).data(), sizeof(double) * a->n);
  });
}

int ref_gram_solve(uint64_t order, const double* w, uint64_t nrhs, const double* rhs, double* x_out,
                   int32_t* used_ldlt, double* pivots_out, char* err, uint64_t errcap) {
  return guarded(err, errcap, [&] {
    Matrix wm(order, order);
    for (std::size_t i = 0; i < order; ++i)
      for (std::size_t j = 0; j < order; ++j) wm(i, j) = w[i * order + j];
    GramSolver g(wm);
    if (used_ldlt) *used_ldlt = g.used_ldlt();
    if (pivots_out)
      for (std::size_t i = 0; i < order; ++i) pivots_out[i] = g.pivots()[i];
    if (nrhs) {
      Matrix r(order, nrhs);
      for (std::size_t i = 0; i < order; ++i)
        for (std::size_t j = 0; j < nrhs; ++j) r(i, j) = rhs[i * nrhs + j];
      Matrix xs = g.solve(r);
      for (std::size_t i = 0; i < order; ++i)
        for (std::size_t j = 0; j < nrhs; ++j) x_out[i * nrhs + j] = xs(i, j);
    }
  });
}

int ref_cholesky_upper(uint64_t order, const double* w, double* r_out, char* err, uint64_t errcap) {
  return guarded(err, errcap, [&] {
    Matrix wm(order, order);
    for (std::size_t i = 0; i < order; ++i)
      for (std::size_t j = 0; j < order; ++j) wm(i, j) = w[i * order + j];
    Matrix r = cholesky_upper(wm);
    for (std::size_t i = 0; i < order; ++i)
      for (std::size_t j = 0; j < order; ++j) r_out[i * order + j] = r(i, j);
  });
}

int ref_hessenberg_lsq(uint64_t rows, uint64_t cols, const double* g, double beta, double* y_out,
                       double* residual_out, char* err, uint64_t errcap) {
  return guarded(err, errcap, [&] {
    Matrix gm(rows, cols);
    for (std::size_t i = 0; i < rows; ++i)
      for (std::size_t j = 0; j < cols; ++j) gm(i, j) = g[i * cols + j];
    LsqSolution s = hessenberg_lsq(gm, beta);
    for (std::size_t i = 0; i < s.y.size(); ++i) y_out[i] = s.y[i];
    if (residual_out) *residual_out = s.residual_norm;
  });
}

int ref_mr_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return mr_solve(op, fs, xv, oconf(cfg)); });
}
int ref_omin_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return omin_solve(op, fs, xv, oconf(cfg)); });
}
int ref_gmres_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return gmres_solve(op, fs, xv, oconf(cfg)); });
}
int ref_smr_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return smr_solve(op, fs, xv, sconf(cfg)); });
}
int ref_somin_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return somin_solve(op, fs, xv, sconf(cfg)); });
}
int ref_sgmres_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep) {
  return run_solver(a, f, x, rep, [&](auto& op, auto fs, auto& xv) { return sgmres_solve(op, fs, xv, sconf(cfg)); });
}

int ref_smr_step(const orc_csr* a, double* x, double* r, uint64_t s, double* coeffs_out, orc_counter* c) {
  return guarded(nullptr, 0, [&] {
    SparseMatrix m = to_sparse(a);
    LinearOperator op = as_operator(m);
    std::vector<double> xv(x, x + a->n), rv(r, r + a->n);
    OpCounter oc;
    std::vector<double> co = smr_step(op, xv, rv, s, &oc);
    std::memcpy(x, xv.data(), sizeof(double) * a->n);
    std::memcpy(r, rv.data(), sizeof(double) * a->n);
    if (coeffs_out) std::memcpy(coeffs_out, co.data(), sizeof(double) * co.size());
    if (c) *c = conv(oc);
  });
}

int ref_arnoldi(const orc_csr* a, const double* v1, uint64_t m, double* h_out, uint64_t* steps_out,
                int32_t* happy_out) {
  return guarded(nullptr, 0, [&] {
    SparseMatrix sm = to_sparse(a);
    LinearOperator op = as_operator(sm);
    ArnoldiResult r = arnoldi(op, std::span<const double>(v1, a->n), m);
    std::memset(h_out, 0, sizeof(double) * (m + 1) * m);
    for (std::size_t i = 0; i < r.h.rows(); ++i)
      for (std::size_t j = 0; j < r.h.cols(); ++j) h_out[i * m + j] = r.h(i, j);
    *steps_out = r.steps;
    *happy_out = r.happy;
  });
}

int ref_sarnoldi(const orc_csr* a, const double* v1, uint64_t s, uint64_t m_blocks, double* blocks_out,
                 double* grams_out, double* hess_out, double* seed_out, double* seed_norm_out,
                 orc_counter* counter, char* err, uint64_t errcap) {
  return guarded(err, errcap, [&] {
    SparseMatrix sm = to_sparse(a);
    LinearOperator op = as_operator(sm);
    OpCounter oc;
    SStepBasis b = sarnoldi(op, std::span<const double>(v1, a->n), s, m_blocks, &oc);
    const std::size_t n = a->n;
    for (std::size_t bi = 0; bi < b.blocks.size(); ++bi)
      for (std::size_t j = 0; j < s; ++j)
        std::memcpy(blocks_out + (bi * s + j) * n, b.blocks[bi].column(j).data(), sizeof(double) * n);
    for (std::size_t bi = 0; bi < b.grams.size(); ++bi)
      for (std::size_t i = 0; i < s; ++i)
        for (std::size_t j = 0; j < s; ++j) grams_out[bi * s * s + i * s + j] = b.grams[bi](i, j);
    for (std::size_t i = 0; i < b.hess.rows(); ++i)
      for (std::size_t j = 0; j < b.hess.cols(); ++j) hess_out[i * b.hess.cols() + j] = b.hess(i, j);
    std::memcpy(seed_out, b.next_seed.data(), sizeof(double) * n);
    *seed_norm_out = b.next_seed_norm;
    if (counter) *counter = conv(oc);
  });
}

// Test-input helpers: the reference's own problem assembly (problem.hpp:138-199, out of
// the hot-path scope but used by its KATs) and the std::mt19937 uniform stream its test
// oracles draw from (tests/support/oracles.hpp:117-133).
int ref_discretize(uint64_t nx, double beta, double gamma, int32_t symmetric, uint64_t** offs,
                   uint64_t** cols, double** vals, double** rhs, double** x0) {
  return guarded(nullptr, 0, [&] {
    ProblemFunctions p = paper_problem(beta, gamma);
    if (symmetric) {
      p.d = [](double, double) { return 0.0; };
      p.e = [](double, double) { return 0.0; };
    }
    DiscretizedProblem prob = assemble(nx, p);
    const std::size_t n = prob.a.rows(), nnz = prob.a.nnz();
    *offs = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (n + 1)));
    *cols = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * nnz));
    *vals = static_cast<double*>(std::malloc(sizeof(double) * nnz));
    *rhs = static_cast<double*>(std::malloc(sizeof(double) * n));
    *x0 = static_cast<double*>(std::malloc(sizeof(double) * n));
    for (std::size_t i = 0; i <= n; ++i) (*offs)[i] = prob.a.row_offsets()[i];
    for (std::size_t i = 0; i < nnz; ++i) {
      (*cols)[i] = prob.a.col_indices()[i];
      (*vals)[i] = prob.a.values()[i];
    }
    for (std::size_t i = 0; i < n; ++i) {
      (*rhs)[i] = prob.rhs[i];
      (*x0)[i] = prob.x0[i];
    }
  });
}

// ---- ILU(0) (ilu0.hpp): factor values in A's pattern (L strict-lower entries, then U
// entries of each row, A's columns being ascending), the apply z = (LU)^{-1} r, and the
// right-preconditioned driver flow of solve_linear (bench.hpp:149-191; bench.hpp itself needs
// <json.hpp> and does not build here, so its few driver lines are restated with the
// reference's own ilu0_factor / right_preconditioned / ilu0_apply / s-step solvers)
int ref_ilu0_factor(const orc_csr* a, double* lu_out, char* err, uint64_t errcap) {
  return guarded(err, errcap, [&] {
    SparseMatrix m = to_sparse(a);
    Ilu0Factors f = ilu0_factor(m);
    const std::size_t n = a->n;
    std::size_t q = 0;
    for (std::size_t i = 0; i < n; ++i) {
      for (std::size_t p = f.l_unit.row_offsets()[i]; p < f.l_unit.row_offsets()[i + 1]; ++p)
        lu_out[q++] = f.l_unit.values()[p];
      for (std::size_t p = f.u_upper.row_offsets()[i]; p < f.u_upper.row_offsets()[i + 1]; ++p)
        lu_out[q++] = f.u_upper.values()[p];
    }
  });
}

static Ilu0Factors factors_from(const orc_csr* a, const double* lu) {
  std::vector<std::tuple<std::size_t, std::size_t, double>> le, ue;
  for (std::size_t i = 0; i < a->n; ++i)
    for (uint64_t p = a->row_offsets[i]; p < a->row_offsets[i + 1]; ++p) {
      if (a->col_indices[p] < i)
        le.emplace_back(i, a->col_indices[p], lu[p]);
      else
        ue.emplace_back(i, a->col_indices[p], lu[p]);
    }
  return {SparseMatrix::from_triplets(a->n, a->n, std::move(le)), SparseMatrix::from_triplets(a->n, a->n, std::move(ue))};
}

void ref_ilu0_apply(const orc_csr* a, const double* lu, const double* r, double* z) {
  Ilu0Factors f = factors_from(a, lu);
  ilu0_apply(f, std::span<const double>(r, a->n), std::span<double>(z, a->n));
}

// method: 0 s-Omin, 1 s-GMRES, 2 GMRES(m); cfg->tol is the driver's threshold
int ref_solve_linear(const orc_csr* a, const double* f, const double* x0, int32_t method, const orc_sstep_cfg* cfg,
                     int32_t precondition, double* x_out, orc_report* rep) {
  return guarded(rep->error, sizeof rep->error, [&] {
    SparseMatrix m = to_sparse(a);
    const std::size_t n = a->n;
    std::span<const double> fs(f, n);
    std::vector<double> x(x0, x0 + n);
    const SStepConfig c = sconf(cfg);
    auto dispatch = [&](const LinearOperator& op, std::span<const double> rhs, std::vector<double>& xv) {
      if (method == 2) {  // the standard GMRES(m) (solvers.hpp:297-359), as bench.hpp:94-108 configures it
        SolverConfig g;
        g.method = Method::gmres;
        g.k = c.k;
        g.m = c.m;
        g.tol = c.tol;
        g.max_iterations = c.max_iterations;
        return gmres_solve(op, rhs, xv, g);
      }
      return method == 0 ? somin_solve(op, rhs, xv, c) : sgmres_solve(op, rhs, xv, c);
    };
    SolveReport r;
    if (precondition) {
      Ilu0Factors fac = ilu0_factor(m);
      LinearOperator op = right_preconditioned(m, fac);
      std::vector<double> r0 = spmv(m, x);
      for (std::size_t i = 0; i < n; ++i) r0[i] = f[i] - r0[i];
      std::vector<double> w(n, 0.0);
      r = dispatch(op, r0, w);
      r.op_counts.matvecs += 1;
      r.op_counts.vec_updates += 1;
      std::vector<double> z = ilu0_apply(fac, w);
      axpy(1.0, z, x);
      r.op_counts.vec_updates += 1;
    } else {
      r = dispatch(as_operator(m), fs, x);
    }
    std::vector<double> ax = spmv(m, x);
    r.op_counts.matvecs += 1;
    for (std::size_t i = 0; i < n; ++i) ax[i] = f[i] - ax[i];
    r.op_counts.vec_updates += 1;
    r.op_counts.termination_dots += 1;
    const double true_norm = norm2(ax);
    r.residual_history.push_back(true_norm);
    r.final_residual = true_norm;
    if (r.converged && true_norm > c.tol) {
      r.converged = false;
      r.breakdown = "recomputed true residual exceeds the threshold";
    }
    std::memcpy(x_out, x.data(), sizeof(double) * n);
    fill(rep, r);
  });
}

// accounting.hpp: kind 0 predicted_omin(a, b, c), 1 predicted_gmres(a, b).gmres,
// 2 predicted_gmres(a, b).sgmres, 3 somin_audit_slack(a), 4 gmres_audit_slack(),
// 5 sgmres_audit_slack(a, b)
void ref_accounting_predict(int32_t kind, uint64_t a, uint64_t b, uint64_t c, orc_counter* out) {
  OpCounter r;
  switch (kind) {
    case 0: r = predicted_omin(a, b, c); break;
    case 1: r = predicted_gmres(a, b).gmres; break;
    case 2: r = predicted_gmres(a, b).sgmres; break;
    case 3: r = somin_audit_slack(a); break;
    case 4: r = gmres_audit_slack(); break;
    default: r = sgmres_audit_slack(a, b); break;
  }
  *out = orc_counter{r.dotprods, r.matvecs, r.vec_updates, r.stored_vectors, r.termination_dots};
}

// audit(rep{op_history, steady_iteration}, predicted, mode 0 exact / 1 bounded / 2 off, slack):
// flags = ok, matvecs_exact, dotprods_exact, updates_exact; diffs joined by '\n'.
void ref_audit(const orc_counter* hist, uint64_t n_hist, uint64_t steady, const orc_counter* predicted,
               int32_t mode, const orc_counter* slack, int32_t* flags, char* diffs, uint64_t cap) {
  auto oc = [](const orc_counter& c) {
    OpCounter o;
    o.dotprods = c.dotprods;
    o.matvecs = c.matvecs;
    o.vec_updates = c.vec_updates;
    o.stored_vectors = c.stored_vectors;
    o.termination_dots = c.termination_dots;
    return o;
  };
  SolveReport rep;
  for (uint64_t i = 0; i < n_hist; ++i) rep.op_history.push_back(oc(hist[i]));
  rep.steady_iteration = steady;
  AuditReport v = audit(rep, oc(*predicted), mode == 0 ? AuditMode::exact : mode == 1 ? AuditMode::bounded : AuditMode::off,
                        oc(*slack));
  flags[0] = v.ok;
  flags[1] = v.matvecs_exact;
  flags[2] = v.dotprods_exact;
  flags[3] = v.updates_exact;
  std::string j;
  for (std::size_t i = 0; i < v.diffs.size(); ++i) j += (i ? "\n" : "") + v.diffs[i];
  if (cap) std::snprintf(diffs, cap, "%s", j.c_str());
}

void ref_free(void* p) { std::free(p); }

void ref_mt_uniform(uint32_t seed, uint64_t count, double lo, double hi, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (uint64_t i = 0; i < count; ++i) out[i] = dist(rng);
}

}  // extern "C"
