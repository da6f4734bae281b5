// Do DMMA (mma.sync f64) and DFMA issue concurrently on sm_100a?  Times a DMMA-only, a
// DFMA-only and a mixed kernel (each warp interleaves both at a given ratio).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NM, int NF>
__global__ void mix(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[4][2] = {};
  double f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NM; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k & 3][0]), "+d"(c[k & 3][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k & 7] = fma(f[k & 7], 0.9999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <int NM, int NF>
int run(double* out, int sms) {
  const int blocks = sms * 8, threads = 256, iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  mix<NM, NF><<<blocks, threads>>>(out, iters);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); mix<NM, NF><<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32 * iters;
  const double tf_mma = 512.0 * NM * warps / (best * 1e-3) / 1e12;
  const double tf_fma = 64.0 * NF * warps / (best * 1e-3) / 1e12;
  printf("{\"dmma_per_iter\": %d, \"dfma_per_iter\": %d, \"ms\": %.4f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
         NM, NF, best, tf_mma, tf_fma, tf_mma + tf_fma);
  return 0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 8));
  run<4, 0>(out, sms); run<0, 32>(out, sms); run<4, 8>(out, sms); run<4, 16>(out, sms); run<4, 32>(out, sms);
  run<2, 16>(out, sms); run<4, 64>(out, sms);
  return 0;
}
