// Dense complex128 linear algebra used on the hot path: a register-tiled FP64
// ZGEMM (the G2 contractions of the apply and the sketch / projection products
// of the TT-cross factorisation) and small elementwise helpers.
//
// Tile 64 x 64 x 8, 256 threads, 4 x 4 complex outputs per thread, smem
// double-buffered through registers; op(A), op(B) in {N, T, C}; batched over up
// to three problems (the chi components) with individual shapes; deterministic
// split-K through a partial workspace.
#include "kernels.cuh"
#include "dmma_tile.cuh"

#include <algorithm>
#include <cstdlib>

namespace vsie {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VSIE_PDL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

int64_t& launch_counter() {
  static thread_local int64_t n = 0;
  return n;
}

namespace {

constexpr int BM = 64, BN = 64, BK = 8, NT = 256;

template <int TA>
__device__ __forceinline__ cplx load_a(const cplx* A, int64_t lda, int64_t M, int64_t K, int64_t m, int64_t k) {
  if (m >= M || k >= K) return cmk(0, 0);
  if (TA == kN) return __ldg(A + m + lda * k);
  cplx v = __ldg(A + k + lda * m);
  if (TA == kC) v.y = -v.y;
  return v;
}
template <int TB>
__device__ __forceinline__ cplx load_b(const cplx* B, int64_t ldb, int64_t K, int64_t N, int64_t k, int64_t n) {
  if (k >= K || n >= N) return cmk(0, 0);
  if (TB == kN) return __ldg(B + k + ldb * n);
  cplx v = __ldg(B + n + ldb * k);
  if (TB == kC) v.y = -v.y;
  return v;
}

template <int TA, int TB>
__global__ void __launch_bounds__(NT) k_zgemm(Zgemm g, int splits, cplx* __restrict__ ws, int64_t ws_stride) {
  const int b = blockIdx.z / splits, sp = blockIdx.z % splits;
  const int64_t M = g.M[b], N = g.N[b], K = g.K[b];
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  if (m0 >= M || n0 >= N) return;
  const int64_t kb0 = ceil_div(K, BK) * sp / splits * BK;
  const int64_t kb1 = std::min<int64_t>(K, ceil_div(K, BK) * (sp + 1) / splits * BK);
  const cplx* __restrict__ A = g.A[b];
  const cplx* __restrict__ B = g.B[b];
  const int64_t lda = g.lda[b], ldb = g.ldb[b];
  __shared__ cplx As[2][BK][BM];
  __shared__ cplx Bs[2][BK][BN];
  const int t = threadIdx.x;
  // load mapping
  int am[2], ak[2], bk[2], bn[2];
  for (int q = 0; q < 2; ++q) {
    const int e = t + NT * q;
    if (TA == kN) { am[q] = e % BM; ak[q] = e / BM; } else { ak[q] = e % BK; am[q] = e / BK; }
    if (TB == kN) { bk[q] = e % BK; bn[q] = e / BK; } else { bn[q] = e % BN; bk[q] = e / BN; }
  }
  cplx ra[2], rb[2];
  auto fetch = [&](int64_t k0) {
    for (int q = 0; q < 2; ++q) {
      ra[q] = load_a<TA>(A, lda, M, kb1, m0 + am[q], k0 + ak[q]);
      rb[q] = load_b<TB>(B, ldb, kb1, N, k0 + bk[q], n0 + bn[q]);
    }
  };
  auto stash = [&](int buf) {
    for (int q = 0; q < 2; ++q) {
      As[buf][ak[q]][am[q]] = ra[q];
      Bs[buf][bk[q]][bn[q]] = rb[q];
    }
  };
  const int tx = t % 16, ty = t / 16;
  cplx acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = cmk(0, 0);
  int buf = 0;
  if (kb0 < kb1) {
    fetch(kb0);
    stash(0);
    __syncthreads();
    for (int64_t k0 = kb0; k0 < kb1; k0 += BK) {
      const bool more = k0 + BK < kb1;
      if (more) fetch(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        cplx av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][tx + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][ty + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) cfma(acc[i][j], av[i], bv[j]);
      }
      if (more) {
        stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  if (splits > 1) {
    cplx* P = ws + ((int64_t)b * splits + sp) * ws_stride;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t m = m0 + tx + 16 * i, n = n0 + ty + 16 * j;
        if (m < M && n < N) P[m + M * n] = acc[i][j];
      }
    return;
  }
  cplx* __restrict__ C = g.C[b];
  const int64_t ldc = g.ldc[b];
  const bool has_beta = g.beta.x != 0.0 || g.beta.y != 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + tx + 16 * i, n = n0 + ty + 16 * j;
      if (m < M && n < N) {
        cplx v = cmul(g.alpha, acc[i][j]);
        if (has_beta) v = cadd(v, cmul(g.beta, C[m + ldc * n]));
        C[m + ldc * n] = v;
      }
    }
}

// C = alpha sum_q ws[q] + beta C over the split-K partials: 8 partial loads in flight per
// thread, summed in a fixed order (deterministic)
__global__ void k_splitk_reduce(Zgemm g, int splits, const cplx* __restrict__ ws, int64_t ws_stride) {
  pdl_wait();
  // tiny kernel: let the next (streaming) kernel launch now, so that it prefetches its
  // constant core while this one runs (it still waits for our completion to read us)
  pdl_trigger();
  const int b = blockIdx.y;
  const int64_t M = g.M[b], N = g.N[b];
  const bool has_beta = g.beta.x != 0.0 || g.beta.y != 0.0;
  const cplx* __restrict__ base = ws + (int64_t)b * splits * ws_stride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * N; e += (int64_t)gridDim.x * blockDim.x) {
    cplx acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = cmk(0, 0);
    int q = 0;
    for (; q + 8 <= splits; q += 8) {
      cplx v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(base + (int64_t)(q + j) * ws_stride + e);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = cadd(acc[j], v[j]);
    }
    for (int j = 0; q < splits; ++q, ++j) acc[j] = cadd(acc[j], __ldcg(base + (int64_t)q * ws_stride + e));
    cplx s = cadd(cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])), cadd(cadd(acc[4], acc[5]), cadd(acc[6], acc[7])));
    const int64_t m = e % M, n = e / M;
    cplx* c = g.C[b] + m + g.ldc[b] * n;
    cplx v = cmul(g.alpha, s);
    if (has_beta) v = cadd(v, cmul(g.beta, *c));
    *c = v;
  }
}

__global__ void k_conj(cplx* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i].y = -x[i].y;
}

__global__ void k_axpy1(const cplx* __restrict__ x, cplx* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = cadd(y[i], x[i]);
}


// ---------------------------------------------------------------------------------------
// Small / skinny ZGEMM on FP64 tensor cores (mma.sync.m8n8k4.f64, SASS DMMA; tcgen05 has
// no f64 kind): a CTA of 4 warps owns a 32 x 32 output tile (warp: 16 x 16 = 2 x 2 DMMA
// tiles, 4 real DMMAs per complex product).  K is walked in chunks of 32: every thread
// loads 8 + 8 elements of the next A / B chunk into registers (coalesced, all in flight)
// while the warps run the current chunk's 8 k-steps out of shared memory.  Padded smem
// rows make both the fragment reads and the stores bank-conflict free.  Deterministic
// split-K through the partial workspace (fixed-order reduction kernel).
__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int TCM = 32, TCN = 32, TCK = 32;
constexpr int TCA = TCM + 2;  // As row stride (complex): 544 B -> fragment reads conflict free
constexpr int TCB = TCK + 4;  // Bs row stride (complex): 576 B

template <int TA>
__global__ void __launch_bounds__(128) k_zgemm_dmma(const __grid_constant__ Zgemm g, int splits, int64_t mt, int64_t nt,
                                                    cplx* __restrict__ ws, int64_t ws_stride) {
  __shared__ cplx As[TCK][TCA];   // As[k][m] = op(A)[m0 + m, kc + k]
  __shared__ cplx Bs[TCN][TCB];   // Bs[n][k] = B[kc + k, n0 + n]
  const int b = blockIdx.y;
  const int64_t tiles = mt * nt;
  const int64_t tile = blockIdx.x % tiles;
  const int sp = (int)(blockIdx.x / tiles);
  const int64_t M = g.M[b], N = g.N[b], K = g.K[b];
  const int64_t m0 = (tile % mt) * TCM, n0 = (tile / mt) * TCN;
  if (m0 >= M || n0 >= N) return;
  const int64_t chunks = (K + TCK - 1) / TCK;
  const int64_t kc0 = chunks * sp / splits * TCK, kc1 = min(K, chunks * (sp + 1) / splits * TCK);
  const cplx* __restrict__ A = g.A[b];
  const cplx* __restrict__ B = g.B[b];
  const int64_t lda = g.lda[b], ldb = g.ldb[b];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 16, wn = (warp >> 1) * 16;
  const int gq = lane >> 2, t = lane & 3;
  cplx ra[8], rb[8];
  auto load = [&](int64_t kc) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 128 * i;
      int mm, kk;
      if (TA == kN) { mm = e & 31; kk = e >> 5; } else { kk = e & 31; mm = e >> 5; }
      const int64_t m = m0 + mm, k = kc + kk;
      cplx v = cmk(0, 0);
      if (m < M && k < kc1) {
        v = TA == kN ? __ldg(A + m + lda * k) : __ldg(A + k + lda * m);
        if (TA == kC) v.y = -v.y;
      }
      ra[i] = v;
      const int kb = e & 31, nb = e >> 5;
      const int64_t n = n0 + nb, k2 = kc + kb;
      rb[i] = (n < N && k2 < kc1) ? __ldg(B + k2 + ldb * n) : cmk(0, 0);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 128 * i;
      if (TA == kN) As[e >> 5][e & 31] = ra[i]; else As[e & 31][e >> 5] = ra[i];
      Bs[e >> 5][e & 31] = rb[i];
    }
  };
  double cr[2][2][2], ci[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0;
  if (kc0 < kc1) load(kc0);
  for (int64_t kc = kc0; kc < kc1; kc += TCK) {
    __syncthreads();
    store();
    __syncthreads();
    if (kc + TCK < kc1) load(kc + TCK);   // next chunk in flight during this chunk's DMMAs
#pragma unroll
    for (int ks = 0; ks < TCK / 4; ++ks) {
      cplx av[2], bv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) av[i] = As[4 * ks + t][wm + 8 * i + gq];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = Bs[wn + 8 * j + gq][4 * ks + t];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma_acc(cr[i][j][0], cr[i][j][1], av[i].x, bv[j].x);
          dmma_acc(cr[i][j][0], cr[i][j][1], -av[i].y, bv[j].y);
          dmma_acc(ci[i][j][0], ci[i][j][1], av[i].x, bv[j].y);
          dmma_acc(ci[i][j][0], ci[i][j][1], av[i].y, bv[j].x);
        }
    }
  }
  const bool has_beta = g.beta.x != 0.0 || g.beta.y != 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int64_t m = m0 + wm + 8 * i + gq, n = n0 + wn + 8 * j + 2 * t + jj;
        if (m >= M || n >= N) continue;
        const cplx acc = cmk(cr[i][j][jj], ci[i][j][jj]);
        if (splits > 1) {
          ws[((int64_t)b * splits + sp) * ws_stride + m + M * n] = acc;
        } else {
          cplx* c = g.C[b] + m + g.ldc[b] * n;
          cplx v = cmul(g.alpha, acc);
          if (has_beta) v = cadd(v, cmul(g.beta, *c));
          *c = v;
        }
      }
}

// 8-warp smem-staged 3M-DMMA tile (dmma_tile.cuh) per CTA; op(A) in {N, T}, op(B) = N.
template <int WA, int WB, bool TA>
__global__ void __launch_bounds__(tc::kThreads) k_zgemm_tc(const __grid_constant__ Zgemm g, int splits, int64_t mt,
                                                           int64_t nt, cplx* __restrict__ ws, int64_t ws_stride,
                                                           int direct) {
  extern __shared__ __align__(16) unsigned char raw[];
  tc::GemmSmem& sm = *reinterpret_cast<tc::GemmSmem*>(raw);
  constexpr int TM = 16 * WA, TN = 16 * WB;
  pdl_wait();
  const int b = blockIdx.y;
  if (b >= g.nbatch) return;
  const int64_t tiles = mt * nt;
  const int64_t tile = blockIdx.x % tiles;
  const int sp = (int)(blockIdx.x / tiles);
  const int64_t M = g.M[b], N = g.N[b], K = g.K[b];
  const int64_t m0 = (tile % mt) * TM, n0 = (tile / mt) * TN;
  if (m0 >= M || n0 >= N) return;
  const int64_t chunks = (K + tc::GKC - 1) / tc::GKC;
  const int64_t k0 = std::min<int64_t>(K, chunks * sp / splits * tc::GKC);
  const int64_t k1 = std::min<int64_t>(K, chunks * (sp + 1) / splits * tc::GKC);
  cplx* C;
  int64_t ldc;
  if (direct) {
    C = g.C[b] + m0 + g.ldc[b] * n0;
    ldc = g.ldc[b];
  } else {
    C = ws + ((int64_t)b * splits + sp) * ws_stride + m0 + M * n0;
    ldc = M;
  }
  tc::gemm_tile<WA, WB, TA>(g.A[b], g.lda[b], g.B[b], g.ldb[b], M, N, m0, n0, k0, k1, sm, C, ldc);
  pdl_trigger();
}

// the scalar (DFMA) ZGEMM for the operand combinations the DMMA kernel does not take
template <int TA, int TB>
void zgemm_t(const Zgemm& g, int splits, dim3 grid, cplx* ws, int64_t stride, cudaStream_t st) {
  k_zgemm<TA, TB><<<grid, NT, 0, st>>>(g, splits, ws, stride);
}

}  // namespace

void launch_zgemm(const Zgemm& g, cplx* ws, int64_t ws_elems, cudaStream_t st) {
  int64_t mt = 0, nt = 0, kmax = 0, mn = 0;
  for (int b = 0; b < g.nbatch; ++b) {
    mt = std::max(mt, ceil_div(g.M[b], BM));
    nt = std::max(nt, ceil_div(g.N[b], BN));
    kmax = std::max(kmax, g.K[b]);
    mn = std::max(mn, g.M[b] * g.N[b]);
  }
  if (mt == 0 || nt == 0) return;
  int splits = 1;
  const int64_t tiles = mt * nt * g.nbatch;
  if (ws != nullptr && tiles < 148 * 2 && kmax >= 8 * BK) {
    splits = (int)std::min<int64_t>(std::min<int64_t>(148 * 4 / tiles, kmax / (4 * BK)), 64);
    while (splits > 1 && (int64_t)splits * mn * g.nbatch > ws_elems) --splits;
    if (splits < 1) splits = 1;
  }
  dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)(g.nbatch * splits));
  const int key = g.ta * 3 + g.tb;
  switch (key) {
    case 0: zgemm_t<kN, kN>(g, splits, grid, ws, mn, st); break;
    case 1: zgemm_t<kN, kT>(g, splits, grid, ws, mn, st); break;
    case 2: zgemm_t<kN, kC>(g, splits, grid, ws, mn, st); break;
    case 3: zgemm_t<kT, kN>(g, splits, grid, ws, mn, st); break;
    case 4: zgemm_t<kT, kT>(g, splits, grid, ws, mn, st); break;
    case 5: zgemm_t<kT, kC>(g, splits, grid, ws, mn, st); break;
    case 6: zgemm_t<kC, kN>(g, splits, grid, ws, mn, st); break;
    case 7: zgemm_t<kC, kT>(g, splits, grid, ws, mn, st); break;
    default: zgemm_t<kC, kC>(g, splits, grid, ws, mn, st); break;
  }
  VSIE_CHECK_LAUNCH();
  if (splits > 1) {
    dim3 rg((unsigned)std::min<int64_t>(ceil_div(mn, 256), 148 * 8), g.nbatch);
    k_splitk_reduce<<<rg, 256, 0, st>>>(g, splits, ws, mn);
    VSIE_CHECK_LAUNCH();
  }
}

void launch_zgemm_dmma(const Zgemm& g, cplx* ws, int64_t ws_elems, cudaStream_t st) {
  VSIE_REQUIRE(g.tb == kN && g.ta != kC, VSIE_ERR_ARG, "zgemm_dmma: op(A) in {N, T}, op(B) = N");
  int64_t mmax = 0, nmax = 0, kmax = 0, mn = 0;
  for (int b = 0; b < g.nbatch; ++b) {
    mmax = std::max(mmax, g.M[b]);
    nmax = std::max(nmax, g.N[b]);
    kmax = std::max(kmax, g.K[b]);
    mn = std::max(mn, g.M[b] * g.N[b]);
  }
  if (mmax == 0 || nmax == 0) return;
  // warp layout: tall (4 x 2 -> 64 x 32) or wide (2 x 4 -> 32 x 64) output tiles
  const bool tall = mmax >= 2 * nmax;
  const int TM = tall ? tc::FTM : tc::ATM, TN = tall ? tc::FTN : tc::ATN;
  const int64_t mt = ceil_div(mmax, TM), nt = ceil_div(nmax, TN);
  const int64_t tiles = mt * nt * g.nbatch;
  const int64_t chunks = ceil_div(kmax, tc::GKC);
  const bool unit = g.alpha.x == 1.0 && g.alpha.y == 0.0 && g.beta.x == 0.0 && g.beta.y == 0.0;
  int splits = 1;
  if (ws != nullptr && tiles < 2 * 148) {
    // few output tiles with a long K (the transpose G2 step, the block-RHS G4 / G3^T
    // products): split K towards two CTAs per SM, each on >= 3 chunks of 16
    splits = (int)std::min<int64_t>(std::min<int64_t>(ceil_div(2 * 148, tiles), std::max<int64_t>(1, chunks / 3)), 64);
    while (splits > 1 && (int64_t)splits * mn * g.nbatch > ws_elems) --splits;
    splits = std::max(splits, 1);
  }
  const int direct = (splits == 1 && unit) ? 1 : 0;
  VSIE_REQUIRE(direct || (ws != nullptr && (int64_t)splits * mn * g.nbatch <= ws_elems), VSIE_ERR_ARG,
               "zgemm_dmma: workspace too small");
  static bool attr = false;
  const size_t smem = sizeof(tc::GemmSmem);
  if (!attr) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_zgemm_tc<tc::FWA, tc::FWB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_zgemm_tc<tc::FWA, tc::FWB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_zgemm_tc<tc::AWA, tc::AWB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_zgemm_tc<tc::AWA, tc::AWB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)(mt * nt * splits), (unsigned)g.nbatch);
  const bool ta = g.ta == kT;
  const dim3 blk(tc::kThreads);
  if (tall) {
    if (ta) launch_pdl(k_zgemm_tc<tc::FWA, tc::FWB, true>, grid, blk, smem, st, g, splits, mt, nt, ws, mn, direct);
    else launch_pdl(k_zgemm_tc<tc::FWA, tc::FWB, false>, grid, blk, smem, st, g, splits, mt, nt, ws, mn, direct);
  } else {
    if (ta) launch_pdl(k_zgemm_tc<tc::AWA, tc::AWB, true>, grid, blk, smem, st, g, splits, mt, nt, ws, mn, direct);
    else launch_pdl(k_zgemm_tc<tc::AWA, tc::AWB, false>, grid, blk, smem, st, g, splits, mt, nt, ws, mn, direct);
  }
  VSIE_CHECK_LAUNCH();
  if (direct) return;
  dim3 rg((unsigned)std::min<int64_t>(ceil_div(mn, 256), 148 * 8), g.nbatch);
  launch_pdl(k_splitk_reduce, rg, dim3(256), 0, st, g, splits, (const cplx*)ws, mn);
  VSIE_CHECK_LAUNCH();
}

void launch_conj(cplx* x, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_conj<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(x, n);
  VSIE_CHECK_LAUNCH();
}

void launch_axpy1(const cplx* x, cplx* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_axpy1<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 8), 256, 0, st>>>(x, y, n);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie
