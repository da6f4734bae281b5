// Complex128 GEMM tile on the FP64 tensor cores (mma.sync.m8n8k4.f64 -> SASS DMMA;
// tcgen05 has no f64 kind), shared by the persistent apply (mega.cu) and the standalone
// ZGEMM of linalg.cu.  256 threads = 8 warps of 16 x 16 outputs laid out WA x WB; K in
// chunks of 16 staged by cp.async (16-B, L2-coherent, zero-filled out of range) into a
// double-buffered padded smem pair; complex products as three real DMMAs (3M).
#pragma once

#include "common.cuh"

namespace vsie {
namespace tc {

constexpr int kThreads = 256;
constexpr int FWA = 4, FWB = 2, AWA = 2, AWB = 4;
constexpr int FTM = 16 * FWA, FTN = 16 * FWB, ATM = 16 * AWA, ATN = 16 * AWB;
constexpr int GKC = 16;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C[m0.., n0..] (or the split partial) = op(A)[m, k] B[k, n] over k in [k0, k1).  8 warps
// of 16 x 16 (WA x WB); K in chunks of 16 staged by cp.async (16-B, L2-coherent, zero
// fill out of range) into a double-buffered padded smem pair, so the next chunk is in
// flight during this chunk's DMMAs without holding registers.  Complex products use
// three real DMMAs (P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi); Re = P1 - P2,
// Im = P3 - P1 - P2).
struct GemmSmem {
  cplx raw[2 * GKC * (ATM + 2) + 2 * ATN * (GKC + 4) > 2 * GKC * (FTM + 2) + 2 * FTN * (GKC + 4)
               ? 2 * GKC * (ATM + 2) + 2 * ATN * (GKC + 4)
               : 2 * GKC * (FTM + 2) + 2 * FTN * (GKC + 4)];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int WA, int WB, bool TA>
__device__ __noinline__ void gemm_tile(const cplx* __restrict__ A, int64_t lda, const cplx* __restrict__ B,
                                       int64_t ldb, int64_t M, int64_t N, int64_t m0, int64_t n0, int64_t k0,
                                       int64_t k1, GemmSmem& sm, cplx* C, int64_t ldc) {
  constexpr int TM = 16 * WA, TN = 16 * WB, SA = TM + 2, SB = GKC + 4;
  cplx* As = sm.raw;                    // [2][GKC][SA]
  cplx* Bs = sm.raw + 2 * GKC * SA;     // [2][TN][SB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % WA) * 16, wn = (warp / WA) * 16;
  const int gq = lane >> 2, t = lane & 3;
  auto issue = [&](int buf, int64_t kc) {
    for (int e = tid; e < TM * GKC; e += kThreads) {
      int mm, kk;
      if (!TA) { mm = e % TM; kk = e / TM; } else { kk = e % GKC; mm = e / GKC; }
      const int64_t m = m0 + mm, k = kc + kk;
      const bool ok = m < M && k < k1;
      cp_async16(As + (buf * GKC + kk) * SA + mm, ok ? (TA ? A + k + lda * m : A + m + lda * k) : A, ok ? 16 : 0);
    }
    for (int e = tid; e < TN * GKC; e += kThreads) {
      const int kk = e % GKC, nn = e / GKC;
      const int64_t n = n0 + nn, k = kc + kk;
      const bool ok = n < N && k < k1;
      cp_async16(Bs + (buf * TN + nn) * SB + kk, ok ? B + k + ldb * n : B, ok ? 16 : 0);
    }
    cp_async_commit();
  };
  double p1[2][2][2], p2[2][2][2], p3[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) p1[i][j][q] = p2[i][j][q] = p3[i][j][q] = 0;
  const int64_t nch = (k1 - k0 + GKC - 1) / GKC;
  __syncthreads();  // smem may still be read by a previous tile
  if (nch > 0) issue(0, k0);
  for (int64_t ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      issue((int)((ch + 1) & 1), k0 + (ch + 1) * GKC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int buf = (int)(ch & 1);
    const int64_t krem = k1 - (k0 + ch * GKC);
    const int nks = (int)(((krem < GKC ? krem : GKC) + 3) / 4);
    const cplx* Ab = As + buf * GKC * SA;
    const cplx* Bb = Bs + buf * TN * SB;
#pragma unroll
    for (int ks = 0; ks < GKC / 4; ++ks) {
      if (ks < nks) {
        cplx av[2], bv[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) av[i] = Ab[(4 * ks + t) * SA + wm + 8 * i + gq];
#pragma unroll
        for (int j = 0; j < 2; ++j) bv[j] = Bb[(wn + 8 * j + gq) * SB + 4 * ks + t];
        double as[2], bs[2];   // the 3M operand sums, once per fragment
#pragma unroll
        for (int i = 0; i < 2; ++i) as[i] = av[i].x + av[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = bv[j].x + bv[j].y;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            dmma(p1[i][j][0], p1[i][j][1], av[i].x, bv[j].x);
            dmma(p2[i][j][0], p2[i][j][1], av[i].y, bv[j].y);
            dmma(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
          }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int64_t m = m0 + wm + 8 * i + gq, n = n0 + wn + 8 * j + 2 * t + jj;
        if (m < M && n < N)
          C[(m - m0) + ldc * (n - n0)] =
              cmk(p1[i][j][jj] - p2[i][j][jj], p3[i][j][jj] - p1[i][j][jj] - p2[i][j][jj]);
      }
}

}  // namespace tc
}  // namespace vsie
