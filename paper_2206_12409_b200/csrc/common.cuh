// Shared device/host helpers of the Z_bc coupling library (sm_100a).
// Product code only — shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>
#include <utility>
#include <vector>

#include "../../include/vsie_coupling.h"

namespace vsie {

struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define VSIE_CHECK_CUDA(expr)                                                                  \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      throw ::vsie::Error(_e == cudaErrorMemoryAllocation ? VSIE_ERR_NOMEM : VSIE_ERR_CUDA,     \
                          std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " +         \
                              __FILE__ + ":" + std::to_string(__LINE__));                      \
    }                                                                                          \
  } while (0)

#define VSIE_CHECK_LAUNCH() do { VSIE_COUNT_LAUNCH(); VSIE_CHECK_CUDA(cudaGetLastError()); } while (0)

#define VSIE_REQUIRE(cond, code, msg)                                 \
  do {                                                                \
    if (!(cond)) throw ::vsie::Error((code), std::string(msg));       \
  } while (0)

// ----------------------------------------------------------------- complex128 as double2
typedef double2 cplx;

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
// acc += a * b  (4 DFMA)
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ----------------------------------------------------------------- device memory
// Device allocations go through a process-wide hook (vsie_set_allocator; default cudaMalloc /
// cudaFree), e.g. the caller's caching allocator (torch.cuda.caching_allocator_alloc).  Each
// buffer remembers the hook that allocated it and is returned through that hook.
struct AllocHook {
  void* (*alloc)(size_t bytes, void* ctx) = nullptr;   // nullptr: cudaMalloc / cudaFree
  void (*free)(void* p, void* ctx) = nullptr;
  void* ctx = nullptr;
};
AllocHook& alloc_hook();                 // the current hook (capi.cpp)
void* dev_alloc_bytes(size_t bytes, AllocHook& used);
void dev_free_bytes(void* p, const AllocHook& used);

// Simple owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  AllocHook hook;   // the hook that allocated p
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), hook(o.hook) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; hook = o.hook; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    p = static_cast<T*>(dev_alloc_bytes(count * sizeof(T), hook));
    n = count;
  }
  // grow-only reallocation (contents not preserved)
  void ensure(size_t count) { if (count > n) alloc(count); }
  void release() {
    if (p) dev_free_bytes(p, hook);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// ----------------------------------------------------------------- launch accounting
// Every launcher of this library increments this counter (one per kernel launch);
// the handle reports the delta over its apply calls (vsie_info.apply_launches).
int64_t& launch_counter();
#define VSIE_COUNT_LAUNCH() (++::vsie::launch_counter())

// ----------------------------------------------------------------- per-kernel timing
struct TimerSlot {
  std::string name;
  int64_t launches = 0;
  double total_ms = 0;
  int64_t bytes = 0, flops = 0;
};

// ----------------------------------------------------------------- programmatic dependent launch
// Kernels of the apply path call pdl_wait() before touching anything their stream
// predecessor wrote and pdl_trigger() once their main loop is done; launched through
// launch_pdl (programmatic stream serialization) the next kernel of a chain is scheduled
// onto SMs while this one drains instead of after it has fully retired.  Both are no-ops
// for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  VSIE_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace vsie
