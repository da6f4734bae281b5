// Host-synchronised communicator for several processes sharing ONE GPU (CUDA IPC): the same
// Comm interface as the NCCL communicator of the slab partition, so every
// multi-process branch of the apply and the cross build runs on a 1-GPU box.
//
// Each rank owns one device exchange buffer exported with cudaIpcGetMemHandle; the handles
// and a sense-reversing barrier live in a POSIX shared-memory segment named by the caller
// (vsie_build_opts.ipc_name, unique per job).  A collective is: copy the rank's contribution
// into its exchange buffer, synchronise the stream, host barrier, read the peers' buffers
// (device-to-device copies or a fixed-order sum kernel), synchronise, host barrier.  No kernel
// ever waits on another process's kernel (the ranks' contexts are time-sliced on the GPU;
// only the host barrier orders them), and the sums run in rank order 0..P-1 (bitwise
// reproducible, equal to the loopback shards' order).  This is a test transport: a box with
// one GPU per rank uses NCCL over NVLink.
#include "comm.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>

#include "common.cuh"

namespace vsie {

namespace {

constexpr int kMaxIpcRanks = 8;
constexpr int kMagic = 0x56534945;   // "VSIE"

struct IpcShared {
  std::atomic<int> ready;
  std::atomic<int> arrive;
  std::atomic<int> generation;
  std::atomic<int> attached;
  int64_t cap[kMaxIpcRanks];
  cudaIpcMemHandle_t handle[kMaxIpcRanks];
};

struct PeerPtrs {
  const double* p[kMaxIpcRanks];
};

__global__ void k_ipc_sum(double* out, PeerPtrs peers, int world, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0;
    for (int r = 0; r < world; ++r) s += peers.p[r][i];
    out[i] = s;
  }
}

class IpcComm : public Comm {
 public:
  IpcComm(const char* name, int rank, int world) : rank_(rank), world_(world), name_(std::string("/vsie_") + name) {
    VSIE_REQUIRE(world >= 1 && world <= kMaxIpcRanks && rank >= 0 && rank < world, VSIE_ERR_ARG,
                 "ipc comm: world must be 1..8");
    for (int r = 0; r < kMaxIpcRanks; ++r) peer_[r] = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
      shm_unlink(name_.c_str());
      fd_ = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      VSIE_REQUIRE(fd_ >= 0, VSIE_ERR_NCCL, "ipc comm: shm_open(create) failed for " + name_);
      VSIE_REQUIRE(ftruncate(fd_, sizeof(IpcShared)) == 0, VSIE_ERR_NCCL, "ipc comm: ftruncate failed");
    } else {
      // wait for the segment and for its final size (mapping a not yet truncated file faults)
      for (;;) {
        if (fd_ < 0) fd_ = shm_open(name_.c_str(), O_RDWR, 0600);
        struct stat stt;
        if (fd_ >= 0 && fstat(fd_, &stt) == 0 && stt.st_size >= (off_t)sizeof(IpcShared)) break;
        VSIE_REQUIRE(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(120), VSIE_ERR_NCCL,
                     "ipc comm: rank 0 never created " + name_);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* p = mmap(nullptr, sizeof(IpcShared), PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
    VSIE_REQUIRE(p != MAP_FAILED, VSIE_ERR_NCCL, "ipc comm: mmap failed");
    sh_ = static_cast<IpcShared*>(p);
    if (rank == 0) {
      new (&sh_->arrive) std::atomic<int>(0);
      new (&sh_->generation) std::atomic<int>(0);
      new (&sh_->attached) std::atomic<int>(0);
      std::memset(sh_->cap, 0, sizeof(sh_->cap));
      sh_->ready.store(kMagic, std::memory_order_release);
    } else {
      while (sh_->ready.load(std::memory_order_acquire) != kMagic) {
        VSIE_REQUIRE(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(120), VSIE_ERR_NCCL,
                     "ipc comm: segment " + name_ + " never initialised");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
    }
    sh_->attached.fetch_add(1);
    barrier();
    if (rank == 0) shm_unlink(name_.c_str());   // every rank is attached: no file left behind
  }

  ~IpcComm() override {
    for (int r = 0; r < world_; ++r)
      if (r != rank_ && peer_[r]) cudaIpcCloseMemHandle(peer_[r]);
    if (buf_) cudaFree(buf_);
    if (sh_) munmap(sh_, sizeof(IpcShared));
    if (fd_ >= 0) close(fd_);
  }

  int world() const override { return world_; }
  int rank() const override { return rank_; }

  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    ensure(n * sizeof(double));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(buf_, buf, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();
    PeerPtrs pp{};
    for (int r = 0; r < world_; ++r) pp.p[r] = static_cast<const double*>(r == rank_ ? buf_ : peer_[r]);
    const unsigned blocks = (unsigned)std::min<size_t>(148 * 8, (n + 255) / 256);
    k_ipc_sum<<<blocks, 256, 0, st>>>(buf, pp, world_, n);
    VSIE_CHECK_LAUNCH();
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();   // nobody refills its exchange buffer while a peer still reads it
  }

  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    if (n == 0) return;
    ensure(n * sizeof(double));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(buf_, send, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();
    for (int r = 0; r < world_; ++r)
      VSIE_CHECK_CUDA(cudaMemcpyAsync(recv + n * r, r == rank_ ? buf_ : peer_[r], n * sizeof(double),
                                      cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();
  }

  void broadcast(void* data, size_t n_bytes, int root, cudaStream_t st) override {
    if (n_bytes == 0) return;
    ensure(n_bytes);
    if (rank_ == root) VSIE_CHECK_CUDA(cudaMemcpyAsync(buf_, data, n_bytes, cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();
    if (rank_ != root) VSIE_CHECK_CUDA(cudaMemcpyAsync(data, peer_[root], n_bytes, cudaMemcpyDeviceToDevice, st));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(st));
    barrier();
  }

 private:
  // sense-reversing barrier on the shared segment (spins with a yield; 300 s timeout)
  void barrier() {
    const int gen = sh_->generation.load(std::memory_order_acquire);
    if (sh_->arrive.fetch_add(1, std::memory_order_acq_rel) == world_ - 1) {
      sh_->arrive.store(0, std::memory_order_relaxed);
      sh_->generation.fetch_add(1, std::memory_order_acq_rel);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    while (sh_->generation.load(std::memory_order_acquire) == gen) {
      if (++spins > 1000) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        VSIE_REQUIRE(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(300), VSIE_ERR_NCCL,
                     "ipc comm: barrier timeout (a peer process is gone)");
      } else {
        sched_yield();
      }
    }
  }

  // collective: every rank calls it with the same byte count (the collectives are symmetric),
  // so all grow their exchange buffers together and re-open the peers' handles
  void ensure(size_t bytes) {
    if (bytes <= cap_) return;
    const size_t cap = std::max(bytes, 2 * cap_);
    barrier();   // peers are done reading the old buffers
    for (int r = 0; r < world_; ++r)
      if (r != rank_ && peer_[r]) {
        VSIE_CHECK_CUDA(cudaIpcCloseMemHandle(peer_[r]));
        peer_[r] = nullptr;
      }
    if (buf_) VSIE_CHECK_CUDA(cudaFree(buf_));
    buf_ = nullptr;
    VSIE_CHECK_CUDA(cudaMalloc(&buf_, cap));
    VSIE_CHECK_CUDA(cudaIpcGetMemHandle(&sh_->handle[rank_], buf_));
    sh_->cap[rank_] = (int64_t)cap;
    barrier();
    for (int r = 0; r < world_; ++r)
      if (r != rank_) {
        VSIE_REQUIRE(sh_->cap[r] == (int64_t)cap, VSIE_ERR_NCCL, "ipc comm: ranks disagree on the buffer size");
        VSIE_CHECK_CUDA(cudaIpcOpenMemHandle(&peer_[r], sh_->handle[r], cudaIpcMemLazyEnablePeerAccess));
      }
    cap_ = cap;
  }

  int rank_, world_;
  std::string name_;
  int fd_ = -1;
  IpcShared* sh_ = nullptr;
  void* buf_ = nullptr;
  size_t cap_ = 0;
  void* peer_[kMaxIpcRanks];
};

}  // namespace

Comm* make_ipc_comm(const char* name, int rank, int world) { return new IpcComm(name, rank, world); }

}  // namespace vsie
