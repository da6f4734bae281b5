// Microbenchmarks for the FP64 roofline denominators that MEASURED_PEAKS.json
// does not carry: DFMA peak, DMMA (mma.sync f64) peak,
// FP64 sincos/sqrt/rcp throughput, and 16-byte-element HBM streaming.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void sincos_kernel(double* out, int iters) {
  double x = 0.1 + threadIdx.x * 1e-4 + blockIdx.x * 1e-6;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(x, &s, &c);
    acc += s * c;
    x += 0.013;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void rsqrt_kernel(double* out, int iters) {
  double x = 1.1 + threadIdx.x * 1e-4;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double r = sqrt(x);
    acc += 1.0 / r;
    x += 0.013;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void read16(const double2* __restrict__ p, size_t n, double* out) {
  double sx = 0, sy = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(p + i);
    sx += v.x; sy += v.y;
  }
  if (sx + sy == 12345.678) out[0] = sx;
}

__global__ void write16(double2* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_double2((double)i, 1.0);
}

__global__ void copy16(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  const int threads = 256;
  const int blocks = sms * 8;
  int iters = 4096;
  float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.9999, 1e-7); }, 5);
  double dfma_tflops = 2.0 * kChains * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;

  int miters = 2048;
  ms = time_ms([&] { dmma_kernel<<<blocks, threads>>>(out, miters); }, 5);
  // m8n8k4: 8*8*4 = 256 FMA per warp-instruction
  double dmma_tflops = 2.0 * 256 * 4.0 * miters * blocks * (threads / 32) / (ms * 1e-3) / 1e12;

  int siters = 1024;
  ms = time_ms([&] { sincos_kernel<<<blocks, threads>>>(out, siters); }, 5);
  double sincos_rate = (double)siters * blocks * threads / (ms * 1e-3);

  ms = time_ms([&] { rsqrt_kernel<<<blocks, threads>>>(out, siters); }, 5);
  double sqrt_rcp_rate = (double)siters * blocks * threads / (ms * 1e-3);

  size_t n = (size_t)1 << 27;  // 2 GiB of double2
  double2 *a, *b;
  CK(cudaMalloc(&a, n * sizeof(double2)));
  CK(cudaMalloc(&b, n * sizeof(double2)));
  CK(cudaMemset(a, 0, n * sizeof(double2)));
  int sblocks = sms * 8;
  ms = time_ms([&] { read16<<<sblocks, 512>>>(a, n, out); }, 10);
  double rd = n * 16.0 / (ms * 1e-3) / 1e9;
  ms = time_ms([&] { write16<<<sblocks, 512>>>(b, n); }, 10);
  double wr = n * 16.0 / (ms * 1e-3) / 1e9;
  ms = time_ms([&] { copy16<<<sblocks, 512>>>(a, b, n); }, 10);
  double cp = 2.0 * n * 16.0 / (ms * 1e-3) / 1e9;

  printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_tflops\": %.2f, \"dmma_f64_tflops\": %.2f, "
         "\"sincos_f64_per_s\": %.4e, \"sqrt_rcp_f64_per_s\": %.4e, "
         "\"read16_gbs\": %.1f, \"write16_gbs\": %.1f, \"copy16_gbs\": %.1f}\n",
         sms, prop.clockRate, dfma_tflops, dmma_tflops, sincos_rate, sqrt_rcp_rate, rd, wr, cp);
  return 0;
}
