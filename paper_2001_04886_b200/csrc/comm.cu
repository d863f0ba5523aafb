// comm.cu -- the two exchanges the row-slab decomposition needs:
//   * allgather of per-rank dot sums (every rank then adds them in rank order, so all ranks
//     hold bit-identical scalars and take identical control decisions);
//   * halo exchange of the first/last rows of a slab with the neighbouring ranks before a
//     matrix-powers sweep.
// Backends: NCCL (dlopen'd libnccl.so.2, stream-ordered, no host synchronization) and a
// host-callback backend (device -> host, caller-provided collective, host -> device) used to
// test the multi-rank data path with several processes sharing one GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "skc_internal.hpp"

namespace skc {

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  // torch ships its own libnccl.so.2; if it is already loaded this returns that instance
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) fail(SKC_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* s) {
    void* p = dlsym(api.h, s);
    if (!p) fail(SKC_ENCCL, std::string("libnccl lacks ") + s);
    return p;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SKC_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclComm : public Comm {
 public:
  NcclComm(int rank, int world, const void* id) {
    this->rank = rank;
    this->world = world;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    nccl_check(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    nccl_check(nccl().AllGather(send, recv, n, ncclDouble, comm_, s), "ncclAllGather");
  }
  void halo(const double* lo_send, double* lo_recv, size_t n_lo, const double* hi_send, double* hi_recv,
            size_t n_hi, cudaStream_t s) override {
    NcclApi& a = nccl();
    nccl_check(a.GroupStart(), "ncclGroupStart");
    if (rank > 0 && n_lo) {
      nccl_check(a.Send(lo_send, n_lo, ncclDouble, rank - 1, comm_, s), "ncclSend");
      nccl_check(a.Recv(lo_recv, n_lo, ncclDouble, rank - 1, comm_, s), "ncclRecv");
    }
    if (rank + 1 < world && n_hi) {
      nccl_check(a.Send(hi_send, n_hi, ncclDouble, rank + 1, comm_, s), "ncclSend");
      nccl_check(a.Recv(hi_recv, n_hi, ncclDouble, rank + 1, comm_, s), "ncclRecv");
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
};

class CallbackComm : public Comm {
 public:
  CallbackComm(int rank, int world, skc_allgather_fn ag, skc_halo_fn hl, void* user)
      : ag_(ag), hl_(hl), user_(user) {
    this->rank = rank;
    this->world = world;
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t s) override {
    std::vector<double> hs(n), hr(n * (size_t)world);
    CK(cudaMemcpyAsync(hs.data(), send, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (ag_(user_, hs.data(), hr.data(), n) != 0) fail(SKC_ENCCL, "allgather callback failed");
    CK(cudaMemcpyAsync(recv, hr.data(), hr.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  void halo(const double* lo_send, double* lo_recv, size_t n_lo, const double* hi_send, double* hi_recv,
            size_t n_hi, cudaStream_t s) override {
    const bool lo = rank > 0 && n_lo, hi = rank + 1 < world && n_hi;
    std::vector<double> ls(lo ? n_lo : 0), lr(lo ? n_lo : 0), hs(hi ? n_hi : 0), hr(hi ? n_hi : 0);
    if (lo) CK(cudaMemcpyAsync(ls.data(), lo_send, n_lo * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (hi) CK(cudaMemcpyAsync(hs.data(), hi_send, n_hi * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hl_(user_, lo ? ls.data() : nullptr, lo ? lr.data() : nullptr, lo ? n_lo : 0, hi ? hs.data() : nullptr,
            hi ? hr.data() : nullptr, hi ? n_hi : 0) != 0)
      fail(SKC_ENCCL, "halo callback failed");
    if (lo) CK(cudaMemcpyAsync(lo_recv, lr.data(), n_lo * sizeof(double), cudaMemcpyHostToDevice, s));
    if (hi) CK(cudaMemcpyAsync(hi_recv, hr.data(), n_hi * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  const char* name() const override { return "callback"; }

 private:
  skc_allgather_fn ag_;
  skc_halo_fn hl_;
  void* user_;
};

}  // namespace

void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof uid);
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id) {
  return std::make_unique<NcclComm>(rank, world, id);
}

std::unique_ptr<Comm> make_callback_comm(int rank, int world, skc_allgather_fn ag, skc_halo_fn hl, void* user) {
  return std::make_unique<CallbackComm>(rank, world, ag, hl, user);
}

// rows [lo, hi) of a slowest dimension of `rows` split over `world` ranks as evenly as possible
void slab_range(int64_t rows, int world, int rank, int64_t& lo, int64_t& hi) {
  lo = rows * rank / world;
  hi = rows * (rank + 1) / world;
}

}  // namespace skc
