/*
 * skrylov_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference s-step Krylov hot path
 * (/root/reference/proj/include/skrylov/{sstep,solvers,small_dense,block,sparse,kernels}.hpp)
 * in plain C, used as the parity checker for the B200 library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it.  The product library (paper_2001_04886_b200/) never links or calls it.
 *
 * The same ABI is exported by oracle/_ref/libskref.so, a thin wrapper compiled
 * directly against the reference headers (oracle/ref_capi.cpp), which pins this
 * restatement bit-for-bit (tests/test_oracle_pin.py).
 *
 * Status codes: 0 ok, 1 invalid_argument, 2 breakdown_error escaped the call,
 * 3 logic_error (debug check), 4 allocation failure.
 */
#ifndef SKRYLOV_ORACLE_H
#define SKRYLOV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t dotprods, matvecs, vec_updates, stored_vectors, termination_dots;
} orc_counter; /* report.hpp:35-41 */

typedef struct {
  uint64_t n;
  const uint64_t* row_offsets; /* n+1 */
  const uint64_t* col_indices; /* nnz, strictly increasing per row */
  const double* values;
} orc_csr; /* sparse.hpp:37-132 (size_t storage) */

typedef struct {
  uint64_t s, k, m;
  double tol;
  uint64_t max_iterations;
  int32_t precondition, unbounded_window, debug_checks;
  double divergence_factor;
} orc_sstep_cfg; /* sstep.hpp:48-58 */

typedef struct {
  int32_t method; /* 0 mr, 1 omin, 2 gcr, 3 gmres (solvers.hpp:41) */
  uint64_t k, m;
  double tol;
  uint64_t max_iterations;
  int32_t precondition, debug_checks;
  double divergence_factor;
} orc_solver_cfg; /* solvers.hpp:45-54 */

typedef struct {
  int32_t converged;
  uint64_t iterations, cycles;
  double* history;
  uint64_t n_history;
  double final_residual;
  orc_counter op_counts;
  orc_counter* op_history;
  uint64_t n_op_history;
  uint64_t steady_iteration;
  int32_t has_breakdown;
  char breakdown[512];
  uint64_t fallback_cycles;
  int32_t n_notes;
  char notes[4][256];
  /* extension (not in SolveReport): per-block-step LSQ residual estimates of s-GMRES */
  double* block_rho;
  uint64_t n_block_rho;
  char error[512]; /* message of a non-zero status */
} orc_report;

/* ILU(0) (ilu0.hpp:39-134): factor values in A's pattern (unit-lower L strictly below the
 * diagonal, U on and above it; A's columns ascending), and z = (LU)^{-1} r */
int orc_ilu0_factor(const orc_csr* a, double* lu_out, char* err, uint64_t errcap);
void orc_ilu0_apply(const orc_csr* a, const double* lu, const double* r, double* z);
/* while set (lu != NULL), every solver applies A (LU)^{-1} for the matrix object `a`
 * (right_preconditioned, ilu0.hpp:138-146); NULL clears it.  Not thread-safe (tests only). */
void orc_set_right_preconditioner(const orc_csr* a, const double* lu);

/* report lifetime */
void orc_report_init(orc_report* r);
void orc_report_free(orc_report* r);

/* kernels.hpp / sparse.hpp */
void orc_spmv(const orc_csr* a, const double* x, double* y);
double orc_dot(uint64_t n, const double* a, const double* b);
/* 0 = reference sequential order (default); 1 = blocked/tree order to measure the envelope */
void orc_set_dot_mode(int mode);
/* 1 = fixed-step benchmark mode: skip the Gram pivot-ratio and LSQ rank aborts (results past
 * them are meaningless); 0 = the reference's behaviour (default) */
void orc_set_fixed_steps(int on);
int orc_krylov_block(const orc_csr* a, const double* v, uint64_t s, double* out /* n*s col-major */);

/* small_dense.hpp: Gram solver (order <= 16). Returns 0 or 2 (breakdown) with message. */
int orc_gram_solve(uint64_t order, const double* w /* row-major */, uint64_t nrhs,
                   const double* rhs /* order x nrhs row-major */, double* x_out,
                   int32_t* used_ldlt, double* pivots_out, char* err, uint64_t errcap);
int orc_cholesky_upper(uint64_t order, const double* w, double* r_out, char* err, uint64_t errcap);
/* one-shot Hessenberg LSQ on a (cols+1) x cols row-major matrix */
int orc_hessenberg_lsq(uint64_t rows, uint64_t cols, const double* g, double beta, double* y_out,
                       double* residual_out, char* err, uint64_t errcap);

/* solvers.hpp */
int orc_mr_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep);
int orc_omin_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep);
int orc_gmres_solve(const orc_csr* a, const double* f, double* x, const orc_solver_cfg* cfg, orc_report* rep);
int orc_arnoldi(const orc_csr* a, const double* v1, uint64_t m, double* h_out /* (m+1) x m */,
                uint64_t* steps_out, int32_t* happy_out);

/* sstep.hpp */
int orc_smr_step(const orc_csr* a, double* x, double* r, uint64_t s, double* coeffs_out, orc_counter* c);
int orc_smr_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep);
int orc_somin_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep);
int orc_sgmres_solve(const orc_csr* a, const double* f, double* x, const orc_sstep_cfg* cfg, orc_report* rep);
/* blocks_out: m_blocks*s*n (block-major, col-major inside), grams_out: m_blocks*s*s,
 * hess_out: ((m_blocks+1)*s) x (m_blocks*s) row-major, seed_out: n. */
int orc_sarnoldi(const orc_csr* a, const double* v1, uint64_t s, uint64_t m_blocks, double* blocks_out,
                 double* grams_out, double* hess_out, double* seed_out, double* seed_norm_out,
                 orc_counter* counter, char* err, uint64_t errcap);

/* Problem generators shared by tests and bench (bit-identical to the product's host generators). */
uint64_t orc_splitmix64(uint64_t* state);
void orc_fill_uniform(uint64_t seed, uint64_t offset, uint64_t n, double* out); /* U[-1,1] */
void orc_fill_lognormal(uint64_t seed, uint64_t n, double* out);               /* exp(N(0,1)) */
/* Assemble the h^2-scaled 5/7-point stencil as CSR in ascending-column order.
 * dim 2: (nx, ny); dim 3: (nx, ny, nz). coef[7] = {-z,-y,-x,C,+x,+y,+z} (2D ignores z).
 * kcell != NULL: variable-diffusion operator with harmonic-mean faces and convection
 * half-coefficient ch2 (coef ignored). Arrays are malloc'ed; free with orc_csr_free. */
int orc_build_stencil_csr(int32_t dim, uint64_t nx, uint64_t ny, uint64_t nz, const double* coef,
                          const double* kcell, double ch2, uint64_t** offs, uint64_t** cols,
                          double** vals);
void orc_csr_free(uint64_t* offs, uint64_t* cols, double* vals);
void orc_stencil_apply(int32_t dim, uint64_t nx, uint64_t ny, uint64_t nz, const double* coef,
                       const double* kcell, double ch2, const double* x, double* y);

#ifdef __cplusplus
}
#endif
#endif
