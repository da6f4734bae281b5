// NCCL communicator loaded with dlopen (per apply, one allreduce
// of 3 r3 values in each direction and one allgather of the m-vector).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace vsie {

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.lib, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.lib, "ncclCommInitRank");
    a.AllReduce = (decltype(a.AllReduce))dlsym(a.lib, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(a.lib, "ncclAllGather");
    a.Broadcast = (decltype(a.Broadcast))dlsym(a.lib, "ncclBroadcast");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.lib, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.lib, "ncclGetErrorString");
  });
  VSIE_REQUIRE(a.lib && a.GetUniqueId && a.CommInitRank && a.AllReduce && a.AllGather && a.CommDestroy,
               VSIE_ERR_NCCL, "libnccl.so.2 not loadable");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw Error(VSIE_ERR_NCCL, std::string(what) + ": " + s);
  }
}

class NcclComm : public Comm {
 public:
  NcclComm(const void* id128, int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId must be 128 bytes");
    std::memcpy(&id, id128, sizeof(id));
    nccl_check(api().CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) api().CommDestroy(comm_);
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    nccl_check(api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    nccl_check(api().AllGather(send, recv, n, ncclFloat64, comm_, st), "ncclAllGather");
  }
  void broadcast(void* buf, size_t n_bytes, int root, cudaStream_t st) override {
    VSIE_REQUIRE(api().Broadcast != nullptr, VSIE_ERR_NCCL, "ncclBroadcast missing");
    nccl_check(api().Broadcast(buf, buf, n_bytes, ncclUint8, root, comm_, st), "ncclBroadcast");
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

Comm* make_nccl_comm(const void* id, int rank, int world) { return new NcclComm(id, rank, world); }

int nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

}  // namespace vsie
