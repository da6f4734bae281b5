// Microbenchmark: raw HBM -> SMEM streaming throughput of cp.async.bulk (1-D TMA) on B200
// with a persistent grid, as a function of stages x piece size and CTAs per SM.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sa(b)), "r"(parity) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar)) : "memory"); }

// each CTA streams its contiguous share; mode 0: thread 0 only (no compute), mode 1: all
// threads read every stage from smem (sum) then sync
__global__ void k_stream(const char* src, int64_t bytes, int stages, int piece, int sub, int mode, double* out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[32];
  const int64_t per = bytes / gridDim.x / piece * piece;
  const char* base = src + per * blockIdx.x;
  const int npieces = (int)(per / piece);
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % stages;
    mbar_expect(&full[s], piece);
    for (int o = 0; o < piece; o += piece / sub) bulk(ring + (size_t)s * piece + o, base + (int64_t)i * piece + o, piece / sub, &full[s]);
  };
  if (threadIdx.x == 0) for (int i = 0; i < stages && i < npieces; ++i) issue(i);
  double acc = 0;
  for (int i = 0; i < npieces; ++i) {
    const int s = i % stages;
    if (mode == 0) {
      if (threadIdx.x == 0) { mbar_wait(&full[s], (i / stages) & 1); if (i + stages < npieces) issue(i + stages); }
    } else {
      mbar_wait(&full[s], (i / stages) & 1);
      const double2* p = (const double2*)(ring + (size_t)s * piece);
      for (int e = threadIdx.x; e < piece / 16; e += blockDim.x) acc += p[e].x;
      __syncthreads();
      if (threadIdx.x == 0 && i + stages < npieces) issue(i + stages);
    }
  }
  if (acc == 1234.5) out[0] = acc;
}
__global__ void k_fill(char* p, size_t n) { for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 16; i += (size_t)gridDim.x * blockDim.x) ((int4*)p)[i] = make_int4(1,2,3,4); }
int main() {
  const int64_t bytes = (int64_t)130 << 20;
  char* src; CK(cudaMalloc(&src, (size_t)1 << 30)); CK(cudaMemset(src, 0, (size_t)1 << 30));
  char* fl; CK(cudaMalloc(&fl, (size_t)512 << 20));
  double* out; CK(cudaMalloc(&out, 8));
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct C { int grid, stages, piece, sub, mode; int64_t bytes; };
  C cs[] = {{148,6,32768,1,0,(int64_t)1 << 30},{148,7,25600,1,0,(int64_t)1 << 30},{148,7,25600,1,1,(int64_t)1 << 30},{296,3,32768,1,0,(int64_t)1 << 30},{296,3,25600,1,0,(int64_t)1 << 30},{296,4,25600,1,0,(int64_t)1 << 30},{296,3,32768,1,1,(int64_t)1 << 30},{296,3,25600,1,1,(int64_t)1 << 30},{444,2,25600,1,0,(int64_t)1 << 30},{444,2,25600,1,1,(int64_t)1 << 30},{148,3,65536,1,0,(int64_t)1 << 30},{148,2,102400,1,0,(int64_t)1 << 30},{296,2,51200,1,0,(int64_t)1 << 30}};
  for (auto c : cs) {
    float best = 1e9, sum = 0; const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      k_fill<<<592, 256>>>(fl, (size_t)512 << 20);
      cudaEventRecord(e0);
      k_stream<<<c.grid, 256, (size_t)c.stages * c.piece>>>(src, c.bytes, c.stages, c.piece, c.sub, c.mode, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 2) { sum += ms; best = ms < best ? ms : best; }
    }
    printf("grid %4d stages %2d piece %6d sub %d mode %d MB %5ld: avg %7.1f us  %6.0f GB/s (best %6.0f)\n", c.grid, c.stages, c.piece, c.sub, c.mode, (long)(c.bytes >> 20),
           sum / reps * 1e3, (double)(c.bytes / c.grid / c.piece * c.piece * c.grid) / (sum / reps * 1e-3) / 1e9, (double)(c.bytes / c.grid / c.piece * c.piece * c.grid) / (best * 1e-3) / 1e9);
  }
  return 0;
}
