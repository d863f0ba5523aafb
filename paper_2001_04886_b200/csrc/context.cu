// context.cu -- context, workspace, profiling, operators and host small-dense helpers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
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
  // at most two co-resident CTAs per SM; each range is a whole number of 256-point tiles
  const int64_t maxg = std::min<int64_t>(2LL * sm_count, kPartialPitch);
  int64_t G = (n + 2047) / 2048;
  G = std::max<int64_t>(1, std::min(G, maxg));
  int64_t range = (n + G - 1) / G;
  range = (range + 255) / 256 * 256;
  G = (n + range - 1) / range;
  g.G = (int)std::max<int64_t>(1, G);
  g.range = range;
  return g;
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
  if (own_stream) cudaStreamDestroy(own_stream);
}

Op::~Op() {
  cudaSetDevice(device);
  for (void* p : owned) cudaFree(p);
}

// ---------------------------------------------------------------- operators
static void* dev_upload(Op& op, const void* host, size_t bytes) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  op.owned.push_back(p);
  if (bytes) CK(cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice));
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
  o.n = o.nx * o.ny * o.nz;
  for (int t = 0; t < 7; ++t) o.coef[t] = d.coef[t];
  o.ch2 = d.ch2;
  if (d.kind == 1) {
    require(kcell_host != nullptr, "stencil: variable-k operator needs the kcell array");
    o.kind = kStencilVarK;
    o.kcell = (const double*)dev_upload(op, kcell_host, sizeof(double) * (size_t)o.n);
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

// ---------------------------------------------------------------- host Hessenberg LSQ
double HessLsq::matrix_norm() const { return std::sqrt(gnorm_sq_); }

double HessLsq::append_column(std::vector<double> col) {
  const size_t j = rcols_.size();
  require(col.size() == j + 2, "hessenberg lsq: column must reach one row below diagonal");
  for (double e : col) gnorm_sq_ += e * e;
  for (size_t t = 0; t < j; ++t) {
    const double a = col[t], b = col[t + 1];
    col[t] = cos_[t] * a + sin_[t] * b;
    col[t + 1] = -sin_[t] * a + cos_[t] * b;
  }
  const double a = col[j], b = col[j + 1];
  const double r = std::hypot(a, b);
  double c = 1.0, s = 0.0;
  if (r != 0.0) {
    c = a / r;
    s = b / r;
  }
  cos_.push_back(c);
  sin_.push_back(s);
  col[j] = r;
  col.pop_back();
  rcols_.push_back(std::move(col));
  rhs_.push_back(0.0);
  const double ra = rhs_[j], rb = rhs_[j + 1];
  rhs_[j] = c * ra + s * rb;
  rhs_[j + 1] = -s * ra + c * rb;
  residual_ = std::fabs(rhs_[j + 1]);
  return residual_;
}

std::vector<double> HessLsq::solve() const {
  const size_t m = rcols_.size();
  const double tol = 1e-14 * matrix_norm();
  std::vector<double> y(m, 0.0);
  for (size_t ii = m; ii-- > 0;) {
    double acc = rhs_[ii];
    for (size_t k = ii + 1; k < m; ++k) acc -= rcols_[k][ii] * y[k];
    if (std::fabs(rcols_[ii][ii]) <= tol)
      fail(SKC_EBREAKDOWN, "hessenberg lsq: rank-deficient R diagonal at column " + std::to_string(ii + 1));
    y[ii] = acc / rcols_[ii][ii];
  }
  return y;
}

}  // namespace skc
