// Cross-GPU combine of the slab partition: NCCL over NVLink /
// NVSwitch, loaded at run time (dlopen, so the library has no link-time NCCL
// dependency and shares torch's already-loaded libnccl.so.2).
#pragma once

#include <cuda_runtime.h>
#include <cstddef>

namespace vsie {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int world() const = 0;
  virtual int rank() const = 0;
  // in-place sum of `n_doubles` doubles across ranks
  virtual void allreduce_sum(double* buf, size_t n_doubles, cudaStream_t st) = 0;
  // recv = concat over ranks of send (n_doubles each)
  virtual void allgather(const double* send, double* recv, size_t n_doubles, cudaStream_t st) = 0;
  // broadcast n bytes of a device buffer from root
  virtual void broadcast(void* buf, size_t n_bytes, int root, cudaStream_t st) = 0;
};

// Several processes on ONE GPU: CUDA-IPC exchange buffers + a host barrier in the POSIX
// shared-memory segment "/vsie_<name>" (comm_ipc.cu; a test transport for 1-GPU boxes).
Comm* make_ipc_comm(const char* name, int rank, int world);
// NCCL communicator; throws Error(VSIE_ERR_NCCL) on failure.
Comm* make_nccl_comm(const void* unique_id_128, int rank, int world);
int nccl_unique_id(void* out128);

}  // namespace vsie
