// context.cu -- context, workspace, profiling, operators and host small-dense helpers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>

#include "skc_internal.hpp"

namespace skc {

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void require(bool ok, const std::string& what) {
  if (!ok) fail(SKC_EINVAL, what);
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e), cudaGetErrorString(e),
                file, line, what);
  fail(e == cudaErrorMemoryAllocation ? SKC_ENOMEM : SKC_ECUDA, buf);
}

std::string fmt_double(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

Geo make_geo(int64_t n, int sm_count) {
  Geo g;
  g.n = n;
  // at most two co-resident CTAs per SM; each range is a whole number of 256-point tiles (small
  // problems spread over up to n / 256 CTAs: a launch-latency-bound sweep then takes one tile
  // round trip instead of a chain of tiles on a few SMs)
  const int64_t maxg = std::min<int64_t>(2LL * sm_count, kPartialPitch);
  int64_t G = (n + 255) / 256;
  G = std::max<int64_t>(1, std::min(G, maxg));
  int64_t range = (n + G - 1) / G;
  range = (range + 255) / 256 * 256;
  G = (n + range - 1) / range;
  g.G = (int)std::max<int64_t>(1, G);
  g.range = range;
  g.cpg = g.G;
  g.gsize = n;
  return g;
}

Geo make_geo_for(const Ctx& c, const Op& op) {
  const int W = c.world();
  const int64_t R = op.d.rows_global > 0 ? op.d.rows_global : op.rows;  // global rows of the slowest dimension
  const int64_t L = op.rowlen > 0 ? op.rowlen : (op.rows > 0 ? op.n / op.rows : 1);
  if (!c.gpu_independent || R % kGroups != 0 || kGroups % W != 0 || L <= 0 || op.d.kind == kIlu0)
    return make_geo(op.n, c.sm_count);
  Geo g;
  g.n = op.n;
  g.gsize = (R / kGroups) * L;
  if (g.gsize * (kGroups / W) != op.n) return make_geo(op.n, c.sm_count);
  // 32 CTAs per group: 2048 partials on one GPU (the pitch), 256 per GPU at 8 GPUs; never below
  // 256 points per CTA
  g.cpg = (int)std::max<int64_t>(1, std::min<int64_t>(32, (g.gsize + 255) / 256));
  int64_t range = (g.gsize + g.cpg - 1) / g.cpg;
  range = (range + 255) / 256 * 256;
  g.cpg = (int)((g.gsize + range - 1) / range);
  g.range = range;
  g.G = (kGroups / W) * g.cpg;
  require(g.G <= kPartialPitch, "grouped geometry: too many partials");
  return g;
}

void ensure_smem_attr(const void* kernel, int bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{kernel, dev}];
  if (have >= bytes) return;
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

// ---------------------------------------------------------------- Ctx
void* Ctx::workspace(const std::string& tag, size_t bytes) {
  auto it = ws.find(tag);
  if (it != ws.end() && it->second.second >= bytes) return it->second.first;
  if (it != ws.end()) {
    CK(cudaStreamSynchronize(stream));
    CK(cudaFree(it->second.first));
    ws.erase(it);
  }
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  ws[tag] = {p, bytes};
  return p;
}

double* Ctx::host_stage(size_t doubles) {
  if (doubles > pinned_cap) {
    if (pinned) CK(cudaFreeHost(pinned));
    pinned_cap = std::max(doubles, pinned_cap * 2);
    CK(cudaMallocHost(&pinned, pinned_cap * sizeof(double)));
  }
  return pinned;
}

int Ctx::prof_begin() {
  if (!profiling) return -1;
  if (event_pool.size() < 2) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      event_pool.push_back(e);
    }
  }
  Pending p;
  p.a = event_pool.back();
  event_pool.pop_back();
  p.b = event_pool.back();
  event_pool.pop_back();
  CK(cudaEventRecord(p.a, stream));
  pending.push_back(p);
  return (int)pending.size() - 1;
}

void Ctx::prof_end(int token, const char* name, double bytes) {
  if (token < 0) return;
  Pending& p = pending[token];
  p.name = name;
  p.bytes = bytes;
  cudaEventRecord(p.b, stream);
}

void Ctx::prof_collect() {
  for (auto& p : pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      KStat& s = stats[p.name];
      s.launches += 1;
      s.ms += ms;
      s.bytes += p.bytes;
    }
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}

void Ctx::sync() {
  CK(cudaStreamSynchronize(stream));
  if (profiling) prof_collect();
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (auto& kv : ws) cudaFree(kv.second.first);
  for (auto e : event_pool) cudaEventDestroy(e);
  for (auto& p : pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  if (pinned) cudaFreeHost(pinned);
  if (aux_stream) {
    cudaStreamSynchronize(aux_stream);
    cudaStreamDestroy(aux_stream);
  }
  if (own_stream) cudaStreamDestroy(own_stream);
}

cudaStream_t Ctx::aux() {
  if (!aux_stream) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&aux_stream, cudaStreamNonBlocking, hi));
  }
  return aux_stream;
}

Op::~Op() {
  cudaSetDevice(device);
  for (void* p : owned) cudaFree(p);
}

// ---------------------------------------------------------------- multi-rank reductions / halos
namespace {
// grouped partials (Geo::enc): per (dot, local group) the sum of its cpg partials in order --
// the first level of reduce_dots_dev's grouped sum -- into out[group * nd + dot]
__global__ void k_local_group_sums(const double* partials, int ngrp, int cpg, int d0, int nd, double* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ngrp * nd; e += gridDim.x * blockDim.x) {
    const int grp = e / nd, d = e % nd;
    const double* p = partials + (int64_t)(d0 + d) * kPartialPitch + (int64_t)grp * cpg;
    double s = 0.0;
    for (int j = 0; j < cpg; ++j) s += p[j];
    out[e] = s;
  }
}
// per-rank sums of dots [d0, d0+nd) over G CTA partials (same fixed order as the scalar kernels)
__global__ void k_local_reduce(const double* partials, int G, int d0, int nd, double* out) {
  for (int d = blockIdx.x; d < nd; d += gridDim.x) {  // one warp per dot, fixed lane order
    const double* p = partials + (int64_t)(d0 + d) * kPartialPitch;
    double s = 0.0;
    for (int g = threadIdx.x; g < G; g += 32) s += p[g];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[d] = s;
  }
}
// recv[r*nd + d] -> partials[(d0+d)*pitch + r]
__global__ void k_scatter_ranks(const double* recv, int world, int nd, double* partials, int d0) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < world * nd; e += gridDim.x * blockDim.x) {
    const int r = e / nd, d = e % nd;
    partials[(int64_t)(d0 + d) * kPartialPitch + r] = recv[e];
  }
}
}  // namespace

int Ctx::reduce_point(double* partials, int G, int d0, int nd) {
  if (!comm || comm->world == 1 || nd <= 0) return G;
  const int W = comm->world;
  constexpr int kRing = 16, kSlot = 32768;
  double* buf = (double*)workspace("reduce_ring", (size_t)kRing * 2 * kSlot * sizeof(double));
  double* send = buf + (size_t)(reduce_ring % kRing) * 2 * kSlot;
  double* recv = send + kSlot;
  ++reduce_ring;
  ++launches;
  if (G >> 16) {  // grouped: allgather each rank's group sums; the kGroups sums, in order, become the partials
    const int Gn = G & 0xffff, cpg = G >> 16, ngl = Gn / cpg;
    require((size_t)ngl * nd <= (size_t)kSlot && (size_t)W * ngl * nd <= (size_t)kSlot,
            "reduce_point: too many dots for one exchange");
    k_local_group_sums<<<std::max(1, std::min(64, (ngl * nd + 255) / 256)), 256, 0, stream>>>(partials, ngl, cpg, d0, nd,
                                                                                            send);
    CK(cudaGetLastError());
    comm->allgather(send, recv, (size_t)ngl * nd, stream);
    ++launches;
    // recv[(r ngl + g) nd + d] = group (r ngl + g)'s sum: partial column r ngl + g
    k_scatter_ranks<<<std::max(1, std::min(64, (W * ngl * nd + 255) / 256)), 256, 0, stream>>>(recv, W * ngl, nd,
                                                                                             partials, d0);
    CK(cudaGetLastError());
    return (W * ngl) | (1 << 16);
  }
  require(nd <= 4096 && (size_t)W * nd <= (size_t)kSlot, "reduce_point: too many dots for one exchange");
  k_local_reduce<<<std::min(nd, 64), 32, 0, stream>>>(partials, G, d0, nd, send);
  CK(cudaGetLastError());
  comm->allgather(send, recv, (size_t)nd, stream);
  ++launches;
  k_scatter_ranks<<<std::max(1, std::min(64, (W * nd + 255) / 256)), 256, 0, stream>>>(recv, W, nd, partials, d0);
  CK(cudaGetLastError());
  return W;
}

void Ctx::halo_exchange(const DevOp& op, const double* v, int J) {
  if (!comm || comm->world == 1 || J <= 0 || op.halo_rows == 0) return;
  require(J <= op.halo_rows, "halo exchange deeper than the operator's halo");
  const int64_t L = op.dim == 2 ? op.nx : op.nx * op.ny;
  const int64_t nrows = op.n / L;
  require(nrows >= J, "slab thinner than the halo width");
  double* hlo = const_cast<double*>(op.hlo);
  double* hhi = const_cast<double*>(op.hhi);
  ++launches;
  comm->halo(v, hlo + (op.halo_rows - J) * L, (size_t)(J * L), v + (nrows - J) * L, hhi, (size_t)(J * L), stream);
}

// ---------------------------------------------------------------- operators
static void* dev_upload(Op& op, const void* host, size_t bytes) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  op.owned.push_back(p);
  if (bytes && host) CK(cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice));
  return p;
}

void build_stencil_op(Ctx& c, Op& op, const skc_stencil_desc& d, const double* kcell_host) {
  require(d.dim == 2 || d.dim == 3, "stencil: dim must be 2 or 3");
  require(d.nx >= 1 && d.ny >= 1 && (d.dim == 2 || d.nz >= 1), "stencil: empty grid");
  require(d.kind == 0 || d.kind == 1, "stencil: kind must be 0 (constant) or 1 (variable k)");
  require(d.nx <= 0x7fffffff && d.ny <= 65535 && (d.dim == 2 || d.nz <= 65535), "stencil: grid too large");
  op.device = c.device;
  DevOp& o = op.d;
  std::memset(&o, 0, sizeof o);
  o.dim = d.dim;
  o.nx = (int64_t)d.nx;
  o.ny = (int64_t)d.ny;
  o.nz = d.dim == 3 ? (int64_t)d.nz : 1;
  for (int t = 0; t < 7; ++t) o.coef[t] = d.coef[t];
  o.ch2 = d.ch2;
  // row slab of the slowest dimension owned by this rank (the whole grid on one GPU)
  const int64_t R = d.dim == 2 ? o.ny : o.nz;
  op.rowlen = d.dim == 2 ? o.nx : o.nx * o.ny;
  int64_t lo = 0, hi = R;
  slab_range(R, c.world(), c.rank(), lo, hi);
  const int64_t H = c.world() > 1 ? kMaxS : 0;
  require(hi - lo >= std::max<int64_t>(H, 1), "stencil slab: fewer rows per rank than the halo width (8)");
  if (d.dim == 2)
    o.ny = hi - lo;
  else
    o.nz = hi - lo;
  o.n = o.nx * o.ny * o.nz;
  o.row0 = lo;
  o.rows_global = R;
  o.halo_rows = H;
  if (H > 0) {
    op.hlo = (double*)dev_upload(op, nullptr, sizeof(double) * (size_t)(H * op.rowlen));
    op.hhi = (double*)dev_upload(op, nullptr, sizeof(double) * (size_t)(H * op.rowlen));
    CK(cudaMemset(op.hlo, 0, sizeof(double) * (size_t)(H * op.rowlen)));
    CK(cudaMemset(op.hhi, 0, sizeof(double) * (size_t)(H * op.rowlen)));
    o.hlo = op.hlo;
    o.hhi = op.hhi;
  }
  if (d.kind == 1) {
    require(kcell_host != nullptr, "stencil: variable-k operator needs the kcell array");
    o.kind = kStencilVarK;
    // k for the owned rows plus H+1 rows each side (clamped to the grid; 1.0 past the edge)
    const int64_t pad = H > 0 ? H + 1 : 0;
    std::vector<double> kp((size_t)((hi - lo + 2 * pad) * op.rowlen), 1.0);
    for (int64_t rr = lo - pad; rr < hi + pad; ++rr)
      if (rr >= 0 && rr < R)
        std::memcpy(kp.data() + (rr - lo + pad) * op.rowlen, kcell_host + rr * op.rowlen,
                    sizeof(double) * (size_t)op.rowlen);
    const double* base = (const double*)dev_upload(op, kp.data(), sizeof(double) * kp.size());
    o.kcell = base + pad * op.rowlen;
    if (d.dim == 3 && c.world() == 1 && c.faces) {
      // every harmonic-mean face once, at setup: the apply then streams them (no divisions)
      double* fc = (double*)dev_upload(op, nullptr, sizeof(double) * 3 * (size_t)o.n);
      launch_faces3(c, o, fc);
      o.faces = fc;
    }
  } else {
    o.kind = kStencilConst;
  }
  op.n = o.n;
  op.rows = o.ny * o.nz;
}

// Recognize a natural-ordering 5/7-point grid pattern in a CSR matrix (no wrap-around).
static bool detect_grid(int64_t n, const uint64_t* offs, const uint64_t* cols, int& dim, int64_t& nx, int64_t& ny,
                        int64_t& nz) {
  std::set<int64_t> d;
  for (int64_t i = 0; i < n; ++i)
    for (uint64_t q = offs[i]; q < offs[i + 1]; ++q) {
      d.insert((int64_t)cols[q] - i);
      if (d.size() > 7) return false;
    }
  std::set<int64_t> absd;
  for (int64_t v : d) absd.insert(v < 0 ? -v : v);
  std::vector<int64_t> pos;
  for (int64_t v : absd)
    if (v > 1) pos.push_back(v);
  int64_t a = 0, b = 0;
  if (pos.empty()) {
    dim = 2;
    nx = n;
    ny = 1;
    nz = 1;
  } else if (pos.size() == 1) {
    a = pos[0];
    if (n % a) return false;
    dim = 2;
    nx = a;
    ny = n / a;
    nz = 1;
  } else if (pos.size() == 2) {
    a = pos[0];
    b = pos[1];
    if (b % a || n % b) return false;
    dim = 3;
    nx = a;
    ny = b / a;
    nz = n / b;
  } else {
    return false;
  }
  for (int64_t v : d) {
    const int64_t av = v < 0 ? -v : v;
    if (!(av == 0 || av == 1 || av == a || (dim == 3 && av == b))) return false;
  }
  // no wrap-around: +-1 stays in the x row, +-nx stays in the plane
  for (int64_t i = 0; i < n; ++i)
    for (uint64_t q = offs[i]; q < offs[i + 1]; ++q) {
      const int64_t j = (int64_t)cols[q], off = j - i;
      if ((off == 1 || off == -1) && (j / nx != i / nx)) return false;
      if (dim == 3 && (off == nx || off == -nx) && (j / (nx * ny) != i / (nx * ny))) return false;
    }
  return true;
}

void validate_csr(int64_t n, const uint64_t* offs, const uint64_t* cols) {
  // sparse.hpp:41-63 invariants
  require(n >= 1, "SparseMatrix: empty matrix");
  require(offs[0] == 0, "SparseMatrix: offsets must start at 0");
  for (int64_t i = 0; i < n; ++i) {
    require(offs[i] <= offs[i + 1], "SparseMatrix: offsets not non-decreasing");
    for (uint64_t q = offs[i]; q < offs[i + 1]; ++q) {
      require(cols[q] < (uint64_t)n, "SparseMatrix: column index out of range");
      require(q == offs[i] || cols[q - 1] < cols[q], "SparseMatrix: columns not strictly increasing within a row");
    }
  }
}

void build_csr_op(Ctx& c, Op& op, int64_t n, const uint64_t* offs, const uint64_t* cols, const double* vals) {
  // sparse.hpp:41-63 invariants
  require(n >= 1, "SparseMatrix: empty matrix");
  require(offs[0] == 0, "SparseMatrix: offsets must start at 0");
  for (int64_t i = 0; i < n; ++i) {
    require(offs[i] <= offs[i + 1], "SparseMatrix: offsets not non-decreasing");
    for (uint64_t q = offs[i]; q < offs[i + 1]; ++q) {
      require(cols[q] < (uint64_t)n, "SparseMatrix: column index out of range");
      require(q == offs[i] || cols[q - 1] < cols[q], "SparseMatrix: columns not strictly increasing within a row");
    }
  }
  require(n <= 0x7fffffff, "csr: n exceeds the int32 column-index range");
  require(c.world() == 1, "csr operators are single-GPU; use skc_op_create_stencil_slab across ranks");
  op.device = c.device;
  DevOp& o = op.d;
  std::memset(&o, 0, sizeof o);
  o.n = n;
  op.n = n;
  int dim = 0;
  int64_t nx = 0, ny = 0, nz = 0;
  if (detect_grid(n, offs, cols, dim, nx, ny, nz) && ny <= 65535 && nz <= 65535) {
    o.kind = kStencilDia;
    o.dim = dim;
    o.nx = nx;
    o.ny = ny;
    o.nz = nz;
    std::vector<double> dia((size_t)7 * n, 0.0);
    const int64_t plane = nx * ny;
    for (int64_t i = 0; i < n; ++i)
      for (uint64_t q = offs[i]; q < offs[i + 1]; ++q) {
        const int64_t off = (int64_t)cols[q] - i;
        int slot = off == 0 ? 3 : off == -1 ? 2 : off == 1 ? 4 : off == -nx ? 1 : off == nx ? 5 : off == -plane ? 0 : 6;
        dia[(size_t)slot * n + i] = vals[q];
      }
    o.dia = (const double*)dev_upload(op, dia.data(), sizeof(double) * dia.size());
    op.rows = ny * nz;
    o.rows_global = dim == 2 ? ny : nz;
    op.rowlen = dim == 2 ? nx : nx * ny;
  } else {
    o.kind = kCsr;
    o.dim = 0;
    std::vector<int64_t> rp(offs, offs + n + 1);
    std::vector<int32_t> ci(offs[n]);
    for (uint64_t q = 0; q < offs[n]; ++q) ci[q] = (int32_t)cols[q];
    o.rowptr = (const int64_t*)dev_upload(op, rp.data(), sizeof(int64_t) * rp.size());
    o.colidx = (const int32_t*)dev_upload(op, ci.data(), sizeof(int32_t) * ci.size());
    o.vals = (const double*)dev_upload(op, vals, sizeof(double) * offs[n]);
    op.rows = n;
  }
}

}  // namespace skc
