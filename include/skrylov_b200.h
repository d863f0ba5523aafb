/*
 * skrylov_b200.h -- C ABI of the B200 s-step Orthomin / s-step GMRES library
 * (libskrylov_b200.so).  Plain C types only: a cgo / JNI / ctypes / Rust binding can
 * bind it directly.  See INTEGRATION.md for the reference-side bindings.
 *
 * Each entry point replaces one reference interface (file:line under
 * /root/reference/proj/include/skrylov/):
 *
 *   skc_somin_solve   <- somin_solve(const LinearOperator&, span f, vector& x, const SStepConfig&)  sstep.hpp:142-143
 *   skc_sgmres_solve  <- sgmres_solve(...same...)                                                   sstep.hpp:493-494
 *   skc_smr_solve     <- smr_solve(...same...)                                                      sstep.hpp:109-110
 *   skc_smr_step      <- smr_step(op, x, r, s, OpCounter*)                                          sstep.hpp:89-91
 *   skc_gmres_solve   <- gmres_solve(op, f, x, const SolverConfig&)  (s=1 path and fallback)        solvers.hpp:297-298
 *   skc_sarnoldi      <- sarnoldi(op, v1, s, m_blocks, OpCounter*) -> SStepBasis                    sstep.hpp:465-467
 *   skc_op_apply      <- LinearOperator::apply(x, y)                                                operator.hpp:43-46
 *   skc_krylov_block  <- krylov_block(op, v, s)                                                     block.hpp:59-67
 *   skc_op_create_csr <- as_operator(const SparseMatrix&)                                           sparse.hpp:155-160
 *   skc_op_create_stencil (new: device-describable 5/7-point operator)
 *   skc_op_create_ilu0 <- right_preconditioned(a, ilu0_factor(a))  (A (LU)^{-1})                 ilu0.hpp:138-146, 45-95
 *   skc_ilu0_solve[_device] <- ilu0_apply(factors, r) -> z = (LU)^{-1} r                         ilu0.hpp:99-134
 *   skc_ilu0_factor   <- ilu0_factor(a) values in A's pattern (factored on ctx's device)           ilu0.hpp:45-95
 *   skc_gram_solve / skc_cholesky_upper / skc_hessenberg_lsq <- GramSolver / cholesky_upper /
 *                      hessenberg_lsq (small_dense.hpp:42-331); host-only, no GPU needed.
 *
 * Error convention (mirrors the reference's exceptions):
 *   SKC_OK                0
 *   SKC_EINVAL            1  std::invalid_argument from require() (kernels.hpp:41-43)
 *   SKC_EBREAKDOWN        2  skrylov::breakdown_error escaping the call (sarnoldi, or a
 *                            Cholesky failure of the first s-GMRES block)
 *   SKC_ELOGIC            3  std::logic_error from debug_checks
 *   SKC_ECUDA             4  CUDA runtime failure (std::runtime_error in the C++ wrapper)
 *   SKC_ENCCL             5  NCCL failure
 *   SKC_ENOMEM            6  device allocation failure
 * Numerical breakdown inside the solvers is NOT an error: it is reported in the report's
 * breakdown string with the reference's prefixes ("basis collapse at setup (",
 * "basis collapse at iteration N (", "divergence: ", "basis collapse (",
 * "invariant subspace reached...").  skc_last_error() returns the message of the last
 * failing call on the calling thread.
 */
#ifndef SKRYLOV_B200_H
#define SKRYLOV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKC_OK 0
#define SKC_EINVAL 1
#define SKC_EBREAKDOWN 2
#define SKC_ELOGIC 3
#define SKC_ECUDA 4
#define SKC_ENCCL 5
#define SKC_ENOMEM 6

typedef struct skc_ctx skc_ctx;
typedef struct skc_op skc_op;
typedef struct skc_report skc_report;

/* report.hpp:35-41 */
typedef struct {
  uint64_t dotprods, matvecs, vec_updates, stored_vectors, termination_dots;
} skc_op_counter;

/* sstep.hpp:48-58 SStepConfig, same field meaning; the reference's defaults are s = 2, k = 2,
 * m = 5, tol = 1e-6, max_iterations = 100000, divergence_factor = 10, flags 0 */
typedef struct {
  uint64_t s, k, m;
  double tol; /* absolute threshold on ||r||_2 */
  uint64_t max_iterations;
  int32_t precondition; /* honored by the driver, not the solvers (sstep.hpp:54): ignored here, as
                         the reference's core loops ignore it; compose ILU(0) right
                         preconditioning with skc_op_create_ilu0 / skc_ilu0_solve */
  int32_t unbounded_window;
  int32_t debug_checks;
  double divergence_factor;
  /* not in the reference: fixed-step benchmark mode.  Nonzero bypasses only the Gram pivot-ratio
   * abort (small_dense.hpp:62-64) and the Hessenberg least-squares rank abort
   * (small_dense.hpp:294-296), so a configuration whose reference run stops there (BASELINE
   * configs 3-5 at s = 8) keeps running the same kernels for max_iterations; results past the
   * point where the reference stops are numerically meaningless.  0 = the reference's behaviour. */
  int32_t fixed_steps;
} skc_sstep_config;

/* solvers.hpp:45-54 SolverConfig, restricted to method = gmres (3) */
typedef struct {
  int32_t method;
  uint64_t k, m;
  double tol;
  uint64_t max_iterations;
  int32_t precondition, debug_checks;
  double divergence_factor;
} skc_solver_config;

/* Device-describable stencil operator (h^2-scaled 5/7-point convection-diffusion).
 * Natural ordering, x fastest. coef = {-z,-y,-x,C,+x,+y,+z} (2D ignores the z slots).
 * kind 0: constant coefficients; kind 1: variable diffusion k per cell (kcell array, n
 * entries, harmonic-mean faces, own k on boundary faces) with convection half-coefficient
 * ch2: lower neighbours -k_f - ch2, upper -k_f + ch2, diagonal sum of the face k_f. */
typedef struct {
  int32_t dim; /* 2 or 3 */
  int32_t kind;
  uint64_t nx, ny, nz;
  double coef[7];
  double ch2;
} skc_stencil_desc;

typedef struct {
  int32_t converged;
  uint64_t iterations, cycles;
  double final_residual;
  skc_op_counter op_counts;
  uint64_t steady_iteration;
  int32_t has_breakdown;
  uint64_t fallback_cycles;
  uint64_t n_history, n_op_history, n_notes, n_block_rho;
} skc_report_summary;

/* ---- library / context ---- */
const char* skc_last_error(void);
const char* skc_version(void);
int skc_device_count(int* count);
/* One context per calling thread (the reference is single-threaded). */
int skc_ctx_create(int device, skc_ctx** out);
int skc_ctx_destroy(skc_ctx* ctx);
/* Use an external CUDA stream (cudaStream_t as uintptr_t, 0 = the context's own). */
int skc_ctx_set_stream(skc_ctx* ctx, uintptr_t stream);
/* Kernel timing: when enabled every hot kernel launch is bracketed by CUDA events on its
 * stream; skc_ctx_kernel_stats returns (launches, total ms, algorithmic bytes) per class. */
int skc_ctx_set_profiling(skc_ctx* ctx, int enable);
int skc_ctx_kernel_stats(skc_ctx* ctx, const char* name, uint64_t* launches, double* total_ms,
                         double* alg_bytes);
int skc_ctx_kernel_names(skc_ctx* ctx, char* buf, size_t cap); /* comma separated */
int skc_ctx_reset_stats(skc_ctx* ctx);
/* Number of device kernel launches issued by the library since the last reset. */
int skc_ctx_launch_count(skc_ctx* ctx, uint64_t* launches);

/* ---- operators ---- */
int skc_op_create_stencil(skc_ctx* ctx, const skc_stencil_desc* desc, const double* kcell_host,
                          skc_op** out);
/* CSR (size_t indices, ascending columns per row; sparse.hpp:37-132).  A 5/7-point grid
 * pattern (column offsets {0,+-1,+-nx[,+-nx*ny]} with no wrap-around) is recognized and
 * run by the stencil kernels from per-cell diagonals; anything else runs the CSR kernel. */
int skc_op_create_csr(skc_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                      const double* values, skc_op** out);
/* ILU(0) right preconditioning, as the reference driver composes it when `precondition` is set
 * (solve_linear, bench.hpp:149-191): the operator A (LU)^{-1} for the solvers (iterate w from 0)
 * and z = (LU)^{-1} w for the update x = x0 + z.  The factorization is the reference's IKJ
 * elimination on pattern(A) (host, same operations and order); errors: a row without a
 * diagonal -> SKC_EINVAL, "ilu0: zero pivot at row N" -> SKC_EBREAKDOWN.  One GPU only.  The
 * triangular solves are bit-identical to ilu0_apply (level-scheduled rows, each row in the
 * reference's order). */
int skc_op_create_ilu0(skc_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                       const double* values, skc_op** out);
int skc_ilu0_solve(skc_ctx* ctx, const skc_op* ilu_op, const double* r, double* z);        /* host buffers */
int skc_ilu0_solve_device(skc_ctx* ctx, const skc_op* ilu_op, const double* r, double* z); /* device, async */
int skc_ilu0_factor(skc_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                    const double* values, double* lu_out);
/* seeded k = exp(N(0,1)) field of the variable-coefficient configurations (BASELINE configs[4];
 * DESIGN.md "Inputs"), host only */
int skc_fill_lognormal(uint64_t seed, uint64_t n, double* out);
/* the paper's test problem, host only (problem.hpp:129-203 discretize(ProblemSpec{nx, beta,
 * gamma}) + initial_guess): CSR (row_offsets n+1; col_indices / values 5n - 4nx, columns
 * ascending), rhs, x0 and (optional, may be NULL) the analytic solution; n = nx^2 */
int skc_discretize(uint64_t nx, double beta, double gamma, uint64_t* row_offsets, uint64_t* col_indices,
                   double* values, double* rhs, double* x0, double* u_true);
int skc_op_destroy(skc_op* op);
int skc_op_size(const skc_op* op, uint64_t* n);
/* 0 = general CSR, 2 = 2D stencil, 3 = 3D stencil, 4 = ILU(0)-preconditioned A (LU)^{-1} */
int skc_op_kind(const skc_op* op, int* kind);
/* y = A x on host buffers (bit-identical to the reference spmv for the same values) */
int skc_op_apply(skc_ctx* ctx, const skc_op* op, const double* x, double* y);
/* [v, A v, ..., A^{s-1} v], out is n*s column-major, host buffers */
int skc_krylov_block(skc_ctx* ctx, const skc_op* op, const double* v, uint64_t s, double* out);

/* ---- reports ---- */
int skc_report_create(skc_report** out);
int skc_report_destroy(skc_report* rep);
int skc_report_get_summary(const skc_report* rep, skc_report_summary* out);
uint64_t skc_report_get_history(const skc_report* rep, double* out, uint64_t cap);
uint64_t skc_report_get_op_history(const skc_report* rep, skc_op_counter* out, uint64_t cap);
/* per-block-step LSQ residual estimates of s-GMRES (extension; not in SolveReport) */
uint64_t skc_report_get_block_rho(const skc_report* rep, double* out, uint64_t cap);
/* copies the string (NUL terminated, truncated to cap) and returns its full length */
uint64_t skc_report_get_breakdown(const skc_report* rep, char* out, uint64_t cap);
uint64_t skc_report_get_note(const skc_report* rep, uint64_t idx, char* out, uint64_t cap);

/* ---- solvers (host buffers: f read, x in/out; all device traffic inside the call) ---- */
int skc_somin_solve(skc_ctx* ctx, const skc_op* op, const double* f, double* x,
                    const skc_sstep_config* cfg, skc_report* rep);
int skc_sgmres_solve(skc_ctx* ctx, const skc_op* op, const double* f, double* x,
                     const skc_sstep_config* cfg, skc_report* rep);
int skc_smr_solve(skc_ctx* ctx, const skc_op* op, const double* f, double* x,
                  const skc_sstep_config* cfg, skc_report* rep);
int skc_gmres_solve(skc_ctx* ctx, const skc_op* op, const double* f, double* x,
                    const skc_solver_config* cfg, skc_report* rep);
/* x, r in/out; coeffs_out (s entries) and counter may be NULL */
int skc_smr_step(skc_ctx* ctx, const skc_op* op, double* x, double* r, uint64_t s, double* coeffs_out,
                 skc_op_counter* counter);
/* Device-resident variants: f_dev / x_dev are device pointers on ctx's device. */
int skc_somin_solve_device(skc_ctx* ctx, const skc_op* op, const double* f_dev, double* x_dev,
                           const skc_sstep_config* cfg, skc_report* rep);
int skc_sgmres_solve_device(skc_ctx* ctx, const skc_op* op, const double* f_dev, double* x_dev,
                            const skc_sstep_config* cfg, skc_report* rep);
/* blocks_out: m_blocks*s*n (block-major, column-major inside); grams_out: m_blocks*s*s;
 * hess_out: ((m_blocks+1)*s) x (m_blocks*s) row-major; seed_out: n. Host buffers. */
int skc_sarnoldi(skc_ctx* ctx, const skc_op* op, const double* v1, uint64_t s, uint64_t m_blocks,
                 double* blocks_out, double* grams_out, double* hess_out, double* seed_out,
                 double* seed_norm_out, skc_op_counter* counter);

/* ---- multi-GPU row-slab decomposition (new -- the reference is single-threaded) ----
 * One process (context) per GPU.  The slowest grid dimension (y in 2D, z in 3D) is split into
 * contiguous slabs, rank r owning global rows [lo, hi) = [R*r/P, R*(r+1)/P).  Solves then take
 * the rank's slab of f and x (the unknowns of rows lo..hi-1, natural order) and every rank
 * returns the same report; ghost rows of width <= 8 are exchanged before each matrix-powers
 * sweep and the per-rank dot sums are allgathered and added in rank order at every reduction.
 * NCCL: rank 0 calls skc_nccl_unique_id, the caller broadcasts the 128 bytes, every rank calls
 * skc_ctx_create_nccl.  The callback backend stages through host memory and lets several
 * processes share one GPU (tests). */
typedef int (*skc_allgather_fn)(void* user, const double* send, double* recv, uint64_t n);
typedef int (*skc_halo_fn)(void* user, const double* lo_send, double* lo_recv, uint64_t n_lo,
                           const double* hi_send, double* hi_recv, uint64_t n_hi);
int skc_nccl_unique_id(void* out128);
int skc_ctx_create_nccl(int device, int rank, int world, const void* id128, skc_ctx** out);
int skc_ctx_create_callback(int device, int rank, int world, skc_allgather_fn allgather, skc_halo_fn halo,
                            void* user, skc_ctx** out);
int skc_ctx_world(const skc_ctx* ctx, int* rank, int* world);
/* GPU-count-independent reductions: every dot product is summed over a fixed tree of 64 row
 * groups of the global grid (rows % 64 == 0), so a solve on 1, 2, 4 or 8 GPUs gives bitwise the
 * same results.  On by default for multi-rank contexts (SKC_PINDEP=0 turns it off); on a single
 * GPU it is opt-in and disables the single-GPU-only kernels (block-iteration kernel, persistent
 * s-Omin) to reproduce the slab results bit for bit.  Not in the reference. */
int skc_ctx_set_gpu_independent(skc_ctx* ctx, int enable);
/* slab of the global stencil owned by ctx's rank; kcell_global (n_global entries) for kind 1 */
int skc_op_create_stencil_slab(skc_ctx* ctx, const skc_stencil_desc* global_desc, const double* kcell_global,
                               uint64_t* row_lo, uint64_t* row_hi, skc_op** out);
/* the partition rule above (pure function, no GPU) */
int skc_slab_range(uint64_t rows, int world, int rank, uint64_t* lo, uint64_t* hi);

/* ---- host small-dense (no GPU needed; the same code runs inside the scalar kernels) ---- */
int skc_gram_solve(uint64_t order, const double* w, uint64_t nrhs, const double* rhs, double* x_out,
                   int32_t* used_ldlt, double* pivots_out);
int skc_cholesky_upper(uint64_t order, const double* w, double* r_out);
int skc_hessenberg_lsq(uint64_t rows, uint64_t cols, const double* g, double beta, double* y_out,
                       double* residual_out);

#ifdef __cplusplus
}
#endif
#endif
