// skc_internal.hpp -- shared types of libskrylov_b200: device operator descriptor,
// streaming-kernel descriptors, the per-thread context and error plumbing.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "../../include/skrylov_b200.h"
#include "small_dense.cuh"

namespace skc {

// ---------------------------------------------------------------- errors
struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void require(bool ok, const std::string& what);  // kernels.hpp:41-43 -> SKC_EINVAL
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define CK(call) ::skc::cuda_check((call), #call, __FILE__, __LINE__)

// ---------------------------------------------------------------- operator
// kIlu0: A (LU)^{-1}, ILU(0) right preconditioning (ilu0.hpp:138-146); host-dispatched only
// (no kernel evaluates it point-wise: applies go through launch_apply)
enum OpKind : int { kCsr = 0, kStencilConst = 1, kStencilVarK = 2, kStencilDia = 3, kIlu0 = 4 };

struct IluData;

// Passed by value to kernels. Natural ordering, x fastest.
struct DevOp {
  int kind;
  int dim;
  int64_t nx, ny, nz, n;
  double coef[7];  // -z,-y,-x,C,+x,+y,+z
  double ch2;
  const double* kcell;   // kStencilVarK
  const double* faces;   // kStencilVarK, 3D on one GPU: the +x | +y | +z face coefficients of every cell (3 n)
  const double* dia;     // kStencilDia: 7 slabs of n values (slot-major), 0 where absent
  const int64_t* rowptr; // kCsr
  const int32_t* colidx;
  const double* vals;
  // row-slab decomposition of the slowest dimension (y in 2D, z in 3D): this rank owns
  // global rows [row0, row0 + local rows); halo_rows ghost rows on each side are received
  // into the operator's halo buffers before a sweep (0 on a single GPU).
  int64_t row0;
  int64_t rows_global;
  int64_t halo_rows;
  const double* hlo;  // halo rows -halo_rows..-1 of the sweep source (valid after an exchange)
  const double* hhi;  // halo rows nrows..nrows+halo_rows-1
  const struct IluData* ilu;  // kIlu0: host-side factors and base operator (never read on device)
};

struct Op {
  DevOp d{};
  int64_t n = 0;
  int64_t rows = 1;      // grid rows (2D: ny, 3D: ny*nz) for reporting
  std::vector<void*> owned;  // device allocations
  int device = 0;
  double* hlo = nullptr;  // halo_rows rows below the slab (rows -halo_rows..-1)
  double* hhi = nullptr;  // halo_rows rows above the slab
  int64_t rowlen = 0;     // points per slowest-dimension row (2D: nx, 3D: nx*ny)
  std::unique_ptr<IluData> ilu;  // kIlu0
  ~Op();
};

// ILU(0) factors on the device (ilu0.hpp:39-134): unit-lower L (strictly below the diagonal)
// and U (on and above) as CSR in A's pattern order, each with a level schedule (rows grouped
// by dependency depth, ascending row index within a level) for the triangular solves
struct IluData {
  Op base;  // A itself (stencil kernels when the pattern is a 5/7-point grid, else CSR)
  int64_t n = 0;
  const int64_t *lrp = nullptr, *urp = nullptr;
  const int32_t *lci = nullptr, *uci = nullptr;
  const double *lv = nullptr, *uv = nullptr;
  const int32_t *lperm = nullptr, *uperm = nullptr;  // rows in level order
  const int64_t *llev = nullptr, *ulev = nullptr;    // level offsets into lperm / uperm
  int nlev_l = 0, nlev_u = 0;
  int64_t nnz_l = 0, nnz_u = 0;
  int64_t maxw_l = 0, maxw_u = 0;  // widest level
  // 2D 5-point grids in natural order: the factors by neighbour (L: S, W; U: C, E, N) with a
  // presence mask per row (the pattern, not the values), for the strip-wavefront solves
  int64_t gnx = 0, gny = 0;         // 0: not a 5-point grid
  const double *lS = nullptr, *lW = nullptr, *uC = nullptr, *uE = nullptr, *uN = nullptr;
  const uint8_t *lm = nullptr, *um = nullptr;
  double* bnd = nullptr;            // per-strip boundary column handed to the next strip
  int* stalled = nullptr;           // set by a strip whose neighbour never delivered (host raises)
};

// ---------------------------------------------------------------- streaming geometry
// Every streaming kernel of a solve uses the same fixed CTA decomposition of [0, n):
// CTA g owns the contiguous range [g*range, min(n,(g+1)*range)) and writes one partial per
// dot, so reductions are deterministic (fixed order, no atomics).
// Grouped (GPU-count-independent) form: the global grid's rows are cut into kGroups equal groups
// (every slab of 1, 2, 4 or 8 ranks is a whole number of them) and each group into cpg CTA
// ranges of `range` points, so CTA b owns [(b / cpg) gsize + (b % cpg) range, ...) of its group
// and every partial covers the same points whatever the GPU count; reductions then sum each
// group's cpg partials in order and the kGroups group sums in order (reduce_dots_dev).
// Ungrouped: cpg = G, gsize = n (CTA b owns [b range, (b+1) range)).
struct Geo {
  int64_t n = 0;
  int G = 1;
  int64_t range = 0;
  int cpg = 1;
  int64_t gsize = 0;
  bool grouped() const { return cpg != G || gsize != n; }
  // the partial count as the reductions take it: G, or G | cpg << 16 for grouped partials
  int enc() const { return grouped() ? (G | (cpg << 16)) : G; }
};
Geo make_geo(int64_t n, int sm_count);
constexpr int kGroups = 64;
struct Op;
struct Ctx;
// the geometry every streaming kernel of a solve on `op` uses: grouped when the context asks
// for GPU-count-independent reductions and the grid qualifies, else make_geo
Geo make_geo_for(const Ctx& c, const Op& op);

constexpr int kThreads = 256;
// every reduction partial lives at partials[dot * kPartialPitch + cta]: kernels with different
// CTA counts can share one partial buffer without overlapping regions
constexpr int kPartialPitch = 2048;

// y_o = base_o [* coef[bscale_o]] + sum_j coef[cbase_j + o] * in_j   (j ascending, o in mask_j)
// then dots over value ids: 0..nout-1 = outputs, nout..nout+nx-1 = extra inputs.
constexpr int LC_MAXIN = 40, LC_MAXOUT = 16, LC_MAXX = 8, LC_MAXD = 64;
struct LinDesc {
  int nin, nout, nx, nd;
  int ncoef;
  const double* in[LC_MAXIN];
  uint16_t mask[LC_MAXIN];
  int16_t cbase[LC_MAXIN];
  double* out[LC_MAXOUT];
  const double* base[LC_MAXOUT];
  int16_t bscale[LC_MAXOUT];
  const double* xin[LC_MAXX];
  uint8_t da[LC_MAXD], db[LC_MAXD];
  const double* coef;  // device coefficient array
  double* partials;    // [(dot0 + d) * G + g]
  int dot0, G;
  int64_t n, range;
  int cpg;             // grouped geometry (Geo): CTAs per group, points per group
  int64_t gsize;
  const int* halt;     // skip when *halt != 0
  const int* cond;     // skip when cond != nullptr && *cond == 0
};

// dots L_l . R_r, dot index (l * nr + r)
constexpr int GR_MAXL = 64, GR_MAXR = 8, GR_LB = 4;
struct GramDesc {
  int nl, nr;
  const double* L[GR_MAXL];
  const double* R[GR_MAXR];
  double* partials;
  int dot0, G;
  // optional per-column output map (mapped != 0): L[l] . R[r] goes to dot rbase[r] + l*rstride[r]
  // and rows l >= lmax[r] are not stored; default: dot0 + l*nr + r
  int mapped;
  int rbase[GR_MAXR], rstride[GR_MAXR], lmax[GR_MAXR];
  int64_t n, range;
  int cpg;
  int64_t gsize;
  const int* halt;
  const int* cond;
};

// ---------------------------------------------------------------- multi-GPU exchanges (comm.cu)
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // every rank sends n doubles, receives world*n (rank-major); stream-ordered
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t s) = 0;
  // lo_* with rank-1, hi_* with rank+1 (skipped at the ends)
  virtual void halo(const double* lo_send, double* lo_recv, size_t n_lo, const double* hi_send, double* hi_recv,
                    size_t n_hi, cudaStream_t s) = 0;
  virtual const char* name() const = 0;
};
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id);
std::unique_ptr<Comm> make_callback_comm(int rank, int world, skc_allgather_fn ag, skc_halo_fn hl, void* user);
void slab_range(int64_t rows, int world, int rank, int64_t& lo, int64_t& hi);

// ---------------------------------------------------------------- context
struct KStat {
  uint64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  // side stream for the latency-bound single-CTA least-squares kernels of s-GMRES, which run
  // beside the next block iteration (created on first use; joined before any result is read)
  cudaStream_t aux_stream = nullptr;
  cudaStream_t aux();
  uint64_t launches = 0;
  bool profiling = false;
  bool pdl = true;   // programmatic dependent launch for solver kernels (SKC_PDL=0 disables)
  bool orth = true;  // on-chip block orthogonalization when it fits (SKC_ORTH=0 disables)
  bool persist = true;  // persistent s-Omin for small problems (SKC_PERSIST=0 disables)
  bool spow = true;     // megakernel: row-streamed candidate powers (SKC_SPOW=0 disables)
  bool bupd = true;     // compile-time-shaped s-Omin half-block update at s > 4 (SKC_BUPD=0: k_upd)
  bool faces = true;    // 3D variable-k apply from face coefficients computed once (SKC_FACES=0: per apply)
  int apply_tma_face = 3;  // stored-face 3D apply through the TMA engine (k_apply3t_face), value = ring slots (SKC_APPLY_TMA_FACE; 0 = the cp.async ring)
  int apply_alt = 0;   // constant 3D apply: alternate launches walk z downwards (1), + evict_first x loads (2) (SKC_APPLY_ALT)
  int apply_flip = 0;  // (the next direction)
  int apply_tma = 3;  // constant 3D stencil: plane tiles through the TMA engine (k_apply3t); SKC_APPLY_TMA = 10 * rows per thread + ring slots, 0 = the cp.async ring
  bool apply_ring = true;  // 3D applies through a shared-memory plane ring (SKC_APPLY_RING=0: z-marching registers)
  // GPU-count-independent reductions (grouped geometry): bitwise the same results on 1, 2, 4
  // or 8 GPUs; on by default across ranks, opt-in on one GPU (SKC_PINDEP=1 /
  // skc_ctx_set_gpu_independent), where it turns the single-GPU-only kernels off
  bool gpu_independent = false;
  bool mpk3 = false;             // one-sweep 3D powers on one GPU (SKC_MPK3=1; slower than the applies so far)
  bool lsq_overlap = true;        // s-GMRES least squares on the side stream (SKC_LSQ_OVERLAP=0: in line)
  bool reorth_host_sync = false;  // slabs: read the reorthogonalization decision back (SKC_REORTH_SYNC=1)
  bool ilu_strips = true;  // ILU(0) on 2D grids: strip-wavefront solves (SKC_ILU_STRIPS=0 disables)
  std::map<std::string, KStat> stats;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  // workspace cache (grows, never shrinks while the context lives)
  std::map<std::string, std::pair<void*, size_t>> ws;
  double* pinned = nullptr;
  size_t pinned_cap = 0;
  std::unique_ptr<Comm> comm;  // null on a single GPU
  int reduce_ring = 0;

  int world() const { return comm ? comm->world : 1; }
  int rank() const { return comm ? comm->rank : 0; }
  // Make the dots [d0, d0+nd) of a partial buffer (written by G CTAs) global: on one GPU a
  // no-op returning G; across ranks the per-rank sums are allgathered and scattered back
  // into the first `world` partial columns, so the scalar kernels read them unchanged.
  int reduce_point(double* partials, int G, int d0, int nd);
  // fill op.hlo / op.hhi with the J rows of v owned by the neighbouring ranks
  void halo_exchange(const DevOp& op, const double* v, int J);

  void* workspace(const std::string& tag, size_t bytes);
  double* host_stage(size_t doubles);
  // profiling bracket around one launch
  int prof_begin();
  void prof_end(int token, const char* name, double bytes);
  void prof_collect();
  void sync();
  ~Ctx();
};

// Kernel launch with programmatic dependent launch: the grid may be scheduled while the
// previous kernel on the stream drains (its CTAs set up, then wait in SKC_PDL_ENTRY until the
// previous grid has completed and its writes are visible), hiding the launch gap.
template <typename... KArgs, typename... Args>
inline void launch_k(Ctx& c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c.pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Raise a kernel's dynamic shared-memory limit to `bytes` on the current device, once per
// (kernel, device): the attribute is per device, so a process-wide flag would leave the second
// GPU of a multi-context process at the 48 KB default.  Thread-safe.
void ensure_smem_attr(const void* kernel, int bytes);
template <typename K>
inline void ensure_smem(K* kernel, size_t bytes) {
  ensure_smem_attr(reinterpret_cast<const void*>(kernel), (int)bytes);
}

// RAII launch bracket
struct Launch {
  Ctx& c;
  int tok;
  const char* name;
  double bytes;
  Launch(Ctx& ctx, const char* nm, double b) : c(ctx), tok(ctx.prof_begin()), name(nm), bytes(b) {
    ++ctx.launches;
  }
  ~Launch() { c.prof_end(tok, name, bytes); }
};

// ---------------------------------------------------------------- kernel launchers (kernels.cu)
void launch_apply(Ctx& c, const DevOp& op, const double* x, double* y, const int* halt, const int* cond);
void launch_lincomb(Ctx& c, const LinDesc& d, const char* name = "lincomb");
void launch_gram(Ctx& c, const GramDesc& d, const char* name = "gram");
void launch_fill(Ctx& c, double* p, double v, int64_t n);
// matrix powers (mpk.cu): out[0..J] of src*scale; products X[x] . level j (j >= jdot0) at
// dot0 + x*(J-jdot0+1) + (j-jdot0) as partials over the returned CTA count.
int mpk_max_depth(const DevOp& op);
// depth to use for a powers sweep: on one GPU the 3D sweep (CTA tile with a J-wide ghost
// zone, one barrier per plane) loses to J single-level applies; slabs need it for the halos
int powers_depth(const Ctx& c, const DevOp& op);
constexpr int kMpkMaxDotDepth = 3;  // deepest sweep that can fuse products (launch_mpk)
enum : uint8_t { kHintNormal = 0, kHintFirst = 1, kHintLast = 2 };  // L2 policies of streamed vectors
// one-sweep 3D powers on one GPU (mpk3.cu): constant 7-point stencil, J <= 4; false when the
// operator / depth does not qualify (the caller then uses launch_mpk or repeated applies)
bool launch_mpk3(Ctx& c, const DevOp& op, const double* src, const double* scale, double* const* out, int J,
                 const int* halt, const int* cond, const char* name = "mpk3");
int launch_mpk(Ctx& c, const DevOp& op, const double* src, const double* scale, double* const* out, int J, int nxd,
               const double* const* X, int jdot0, double* partials, int dot0, const int* halt, const int* cond,
               const char* name = "mpk");
// One block-MGS round of s-step Arnoldi (Scalar2 + update, sstep.hpp:338-353).  The kernel
// prologue is the round's scalar step, computed redundantly by every CTA: reduce the incoming
// products V_i^T cand[:,1:] (partials `src` rows src_d0.., src_G columns, fixed order), solve
// W_i t = (V_i^T cand) with block i's Gram factor; CTA 0 records t into rec_t (row l, column
// jc at l*s + jc; added to the stored value on the reorthogonalization pass).  Then
// cand[:,jc] -= sum_l t(l,jc-1) V_i[:,l], fused with the next round's products
// Vnext[l] . cand[jc] at dot0 + l*(s-1) + jc-1 when Vnext is given.
struct MgsScalar {
  const double* src;
  int src_G, src_d0;
  const Gram* gram;
  double* rec_t;
  int accumulate;
  int full;  // the products are a full s x s block [l][jc] (block 0 of the cross products), not [l][jc-1]
};
void launch_mgs(Ctx& c, const Geo& geo, int s, const double* const* Vi, double* const* cand, const double* const* Vnext,
                const MgsScalar& sc, double* partials, int dot0, const int* halt, const int* cond,
                const char* name = "mgs_update");
// operator helpers
void build_stencil_op(Ctx& c, Op& op, const skc_stencil_desc& d, const double* kcell_host);
void launch_faces3(Ctx& c, const DevOp& op, double* faces);
void build_csr_op(Ctx& c, Op& op, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals);
void validate_csr(int64_t n, const uint64_t* offs, const uint64_t* cols);  // sparse.hpp:41-63
// ILU(0) right preconditioning (ilu.cu): op = A (LU)^{-1}; z = (LU)^{-1} r
void build_ilu0_op(Ctx& c, Op& op, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals);
void ilu0_factor_device(Ctx& c, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals,
                        std::vector<double>& lu);
void launch_ilu0_solve(Ctx& c, const IluData& d, const double* r, double* z, const int* halt, const int* cond);
void ilu0_check(Ctx& c, const Op& op);  // raises SKC_ECUDA if a strip solve stalled

// ---------------------------------------------------------------- reports (host)
struct Report {
  bool converged = false;
  uint64_t iterations = 0, cycles = 0;
  std::vector<double> history;
  double final_residual = 0.0;
  skc_op_counter op_counts{};
  std::vector<skc_op_counter> op_history;
  uint64_t steady_iteration = 0;
  std::optional<std::string> breakdown;
  uint64_t fallback_cycles = 0;
  std::vector<std::string> notes;
  std::vector<double> block_rho;
};

struct SStepCfg {
  uint64_t s = 2, k = 2, m = 5;
  double tol = 1e-6;
  uint64_t max_iterations = 100000;
  bool precondition = false, unbounded_window = false, debug_checks = false;
  double divergence_factor = 10.0;
  bool fixed_steps = false;  // benchmark mode: skip the Gram pivot-ratio and LSQ rank aborts
};

// solver entry points (device pointers f, x)
void somin_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep);
void smr_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep);
void sgmres_device(Ctx& c, const Op& op, const double* f, double* x, const SStepCfg& cfg, Report& rep);
void gmres_device(Ctx& c, const Op& op, const double* f, double* x, uint64_t m, double tol,
                  uint64_t max_iterations, Report& rep);
struct BasisOut {
  std::vector<double> blocks, grams, hess, seed;
  double seed_norm = 0.0;
  skc_op_counter counter{};
};
void sarnoldi_device(Ctx& c, const Op& op, const double* v1_dev, uint64_t s, uint64_t m_blocks, BasisOut& out);
void smr_step_device(Ctx& c, const Op& op, double* x, double* r, uint64_t s, double* coeffs,
                     skc_op_counter* counter);

std::string fmt_double(double v);  // std::to_string(double)

}  // namespace skc
