// TMA-streamed GEMVs on the third TT core, batched over the three chi components:
//   forward  (Eq. 17 step 2):      Y3 = G3 y4       (op N, (r2 n3) x r3 times r3)
//   transpose (Eq. 19 step 3):     z3 = G3^T W2     (op T)
// G3^chi is column-major (r2 n3) x r3, one contiguous 28-100 MB stream per
// chi.  Every CTA owns the same fraction [R s / ns, R (s + 1) / ns) of the rows of every chi
// (L <= 32 NQ rows), so that in op N each output row is produced by exactly one CTA (no
// partials) and in op T the CTA's partial z3 is one short vector.  The CTA's row block is a
// set of column segments (16 L bytes each), stored contiguously by the row-blocked copy of
// the core (Shard::G3b; with the canonical layout the 848-B segments cost one bulk copy
// each and the stream ran at 2 TB/s), streamed by a producer warp with one cp.async.bulk
// per stage into a 16-slot ring of <= 10 KB stages; stage i is
// consumed by warp i % 8 alone (lane l: rows l + 32 q of each segment).  op N keeps the
// row accumulators in registers and reduces the 8 warps by a fixed-order smem tree at the
// end of each chi; op T reduces each column pair across the warp (tma::pair_reduce) into a
// per-CTA smem vector written once per chi as the CTA's partial (summed over CTAs in fixed
// order by k_sum_partials_warp).  Deterministic, no atomics.
#include "common.cuh"
#include "kernels.cuh"
#include "tma_ring.cuh"

namespace vsie {
namespace {
using namespace tma;

constexpr int kCW = 8;                      // consumer warps
constexpr int kSegThreads = 32 * (kCW + 1);
constexpr int kStage = 10240;

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kCW) : "memory"); }

// M: 1 op N (x -> y), 2 op T (xt -> yt through partials), 3 both from ONE pass over the core.
// SL ring slots (16: 160 KB, one CTA per SM; 8: 80 KB, leaves room beside it for the CTAs of
// a concurrent compute kernel)
template <int NQ, int M, int SL>
__global__ void __launch_bounds__(kSegThreads, 1) k_seg_gemv(const __grid_constant__ SegGemv a) {
  constexpr int kSlotsS = SL;
  constexpr int kRing = SL * kStage;
  constexpr bool FW = (M & 1) != 0, OPT = (M & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  cplx* ring = reinterpret_cast<cplx*>(smem);
  cplx* red = reinterpret_cast<cplx*>(smem + kRing);   // [4][32 NQ]      (op N)
  cplx* vec = red + (FW ? 4 * 32 * NQ : 0);             // [Cmax]: partial z (op T)
  cplx* vecx = vec + (OPT ? a.cmax : 0);                // [Cmax]: x (op N)
  __shared__ uint64_t full[kSlotsS], empty[kSlotsS];
  const int ns = gridDim.x, s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r0[3], L[3], seg[3], nst[3], off[3];
  int total = 0;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    r0[b] = L[b] = 0;
    seg[b] = 1;
    nst[b] = 0;
    off[b] = total;
    if (b < a.nbatch) {
      const int64_t R = a.R[b];
      r0[b] = (int)(R * s / ns);
      L[b] = (int)(R * (s + 1) / ns) - r0[b];
      seg[b] = L[b] > 0 ? max(1, kStage / (16 * L[b])) : 1;   // column segments per stage
      nst[b] = L[b] > 0 ? (int)((a.C[b] + seg[b] - 1) / seg[b]) : 0;
      total += nst[b];
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlotsS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCW) {
    // producer: G3 is a constant core -- the ring fills before the stream predecessor ends
    if (lane == 0) {
      int i = 0;
      for (int b = 0; b < a.nbatch; ++b) {
        const uint32_t sb = (uint32_t)(16 * L[b]);
        for (int t = 0; t < nst[b]; ++t, ++i) {
          const int slot = i % kSlotsS;
          if (i >= kSlotsS) mbar_wait(&empty[slot], ((i / kSlotsS) - 1) & 1);
          const int cb = t * seg[b];
          const int ncol = (int)min((int64_t)seg[b], a.C[b] - cb);
          mbar_expect_tx(&full[slot], sb * ncol);
          // the block's columns cb .. cb + ncol are one contiguous run of the blocked layout
          bulk_g2s(ring + (size_t)slot * (kStage / 16), a.A[b] + a.C[b] * r0[b] + (int64_t)L[b] * cb, sb * ncol,
                   &full[slot]);
        }
      }
    }
    pdl_wait();
    return;
  }

  pdl_wait();   // x (op N: y4) / w (op T: W2) come from the stream predecessor
  for (int b = 0; b < a.nbatch; ++b) {
    const int Lb = L[b], C = (int)a.C[b];
    const int last = Lb - 1 - lane;
    cplx acc[NQ], w[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      acc[q] = cmk(0, 0);
      w[q] = cmk(0, 0);   // rows past L: zero weight
    }
    if (OPT) {
      const int np = a.xparts[b];
      if (np > 0) {
        // split-K partials of W2: all NQ x 8 loads of a group in flight, fixed summation order
        constexpr int PB = NQ > 4 ? 2 : 8;
        for (int j0 = 0; j0 < np; j0 += PB) {
          cplx v[NQ][PB];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int r = min(lane + 32 * q, Lb - 1);
            const cplx* p = a.xpart[b] + r0[b] + r;
#pragma unroll
            for (int j = 0; j < PB; ++j) v[q][j] = j0 + j < np ? __ldcg(p + a.xpart_stride[b] * (j0 + j)) : cmk(0, 0);
          }
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int j = 0; j < PB; ++j) w[q] = cadd(w[q], v[q][j]);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (lane + 32 * q >= Lb) w[q] = cmk(0, 0);
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = lane + 32 * q;
          if (r < Lb) w[q] = __ldcg(a.xt[b] + r0[b] + r);
        }
      }
    }
    if (FW) {
      // x of this chi (r3 <= ~2k values): a thread's loads in flight before its stores
      for (int c0 = threadIdx.x; c0 < C; c0 += 4 * 32 * kCW) {
        cplx v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 * kCW;
          v[q] = c < C ? __ldcg(a.x[b] + c) : cmk(0, 0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (c0 + q * 32 * kCW < C) vecx[c0 + q * 32 * kCW] = v[q];
      }
    }
    csync();
    if (Lb > 0) {
      for (int t = (warp - off[b] % kCW + kCW) % kCW; t < nst[b]; t += kCW) {
        const int i = off[b] + t;
        const int slot = i % kSlotsS;
        const int cb = t * seg[b];
        const int ncol = min(seg[b], C - cb);
        mbar_wait(&full[slot], (i / kSlotsS) & 1);
        const cplx* st = ring + (size_t)slot * (kStage / 16);
        if (OPT) {
          for (int j = 0; j < ncol; j += 2) {
            const bool two = j + 1 < ncol;
            const cplx* col = st + Lb * j;
            const cplx* col1 = two ? col + Lb : col;
            const cplx xv0 = FW ? vecx[cb + j] : cmk(0, 0), xv1 = FW && two ? vecx[cb + j + 1] : cmk(0, 0);
            cplx d0 = cmk(0, 0), d1 = cmk(0, 0);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const int r = min(32 * q, last) + lane;
              const cplx v0 = col[r], v1 = col1[r];
              cfma(d0, v0, w[q]);
              cfma(d1, v1, w[q]);
              if (FW) {
                cfma(acc[q], v0, xv0);
                cfma(acc[q], v1, xv1);
              }
            }
            const cplx d = pair_reduce(d0, d1, lane);
            if ((lane & 15) == 0 && (lane == 0 || two)) vec[cb + j + (lane >> 4)] = d;
          }
        } else {
          for (int j = 0; j < ncol; ++j) {
            const cplx* col = st + Lb * j;
            const cplx xv = vecx[cb + j];
#pragma unroll
            for (int q = 0; q < NQ; ++q) cfma(acc[q], col[min(32 * q, last) + lane], xv);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
    }
    if (OPT) {
      csync();   // vec complete
      cplx* out = a.partials + ((int64_t)b * ns + s) * a.rstride;
      for (int c = threadIdx.x; c < C; c += 32 * kCW) out[c] = Lb > 0 ? vec[c] : cmk(0, 0);
      csync();   // vec is rewritten by the next chi
    }
    if (FW) {
#pragma unroll
      for (int half = kCW / 2; half >= 1; half >>= 1) {
        if (warp >= half && warp < 2 * half) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) red[(warp - half) * 32 * NQ + lane + 32 * q] = acc[q];
        }
        csync();
        if (warp < half) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q] = cadd(acc[q], red[warp * 32 * NQ + lane + 32 * q]);
        }
        csync();
      }
      if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = lane + 32 * q;
          if (r < Lb) a.y[b][r0[b] + r] = acc[q];
        }
      }
    }
  }
  pdl_trigger();
}

template <int M, int SL>
bool launch_seg(const SegGemv& a, int ns, int nq, size_t smem, cudaStream_t st) {
  switch (nq) {
#define VSIE_SEG(K)                                                                                  \
  case K: {                                                                                          \
    static size_t attr = 0;                                                                          \
    if (smem > attr) {                                                                               \
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_seg_gemv<K, M, SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      attr = smem;                                                                                   \
    }                                                                                                \
    launch_pdl(k_seg_gemv<K, M, SL>, dim3(ns), dim3(kSegThreads), smem, st, a);                      \
    return true;                                                                                     \
  }
    VSIE_SEG(1) VSIE_SEG(2) VSIE_SEG(3) VSIE_SEG(4) VSIE_SEG(5) VSIE_SEG(6) VSIE_SEG(7) VSIE_SEG(8)
    VSIE_SEG(10) VSIE_SEG(12) VSIE_SEG(16)
#undef VSIE_SEG
    default: return false;
  }
}

// shared memory of a launch: ring of SL stages + the op N tree and x (mode 1) and / or the op T
// partial vector (mode 2); SL = 16, 12 or 8 slots, the largest that fits (0: none fits)
int seg_slots(int nq, int64_t cmax, int mode, bool small_ring, size_t* smem_out) {
  const size_t extra = ((mode & 1) ? (size_t)4 * 32 * nq * sizeof(cplx) + (size_t)cmax * sizeof(cplx) : 0) +
                       ((mode & 2) ? (size_t)cmax * sizeof(cplx) : 0);
  for (int sl : {16, 12, 8}) {
    if (small_ring && sl > 8) continue;
    const size_t smem = (size_t)sl * kStage + extra;
    if (smem <= 220 * 1024) {
      *smem_out = smem;
      return sl;
    }
  }
  return 0;
}

int seg_nq(int64_t L) {
  int nq = (int)ceil_div(L, 32);
  if (nq > 8) nq = nq <= 10 ? 10 : nq <= 12 ? 12 : 16;
  return nq;
}

}  // namespace

bool seg_gemv_supported(int64_t R, int64_t C, int nsb) {
  if (R <= 0 || C <= 0 || nsb < 1) return false;
  const int64_t L = ceil_div(R, nsb);
  if (L > 512 || 16 * L > kStage) return false;
  size_t smem = 0;
  return seg_slots(seg_nq(L), C, 3, false, &smem) > 0;
}

// mode 1: op N (x -> y); 2: op T (x -> y through partials); 3: both from one pass
// (op N x -> y, op T xt -> yt)
bool launch_seg_gemv_mode(const SegGemv& a0, int mode, cudaStream_t st, bool small_ring) {
  SegGemv a = a0;
  if (mode == 2)
    for (int b = 0; b < a.nbatch; ++b) {
      a.xt[b] = a0.x[b];
      a.yt[b] = a0.y[b];
    }
  int64_t rmax = 0, cmax = 0;
  for (int b = 0; b < a.nbatch; ++b) {
    rmax = std::max(rmax, a.R[b]);
    cmax = std::max(cmax, a.C[b]);
  }
  if (rmax == 0 || cmax == 0) return false;
  const int ns = a.nsb;
  if (ns < 1) return false;
  const int64_t L = ceil_div(rmax, ns);
  if (L > 512 || 16 * L > kStage) return false;
  const int nq = seg_nq(L);
  a.cmax = cmax;
  size_t smem = 0;
  const int sl = seg_slots(nq, cmax, mode, small_ring, &smem);
  if (sl == 0) return false;
  if (mode & 2) VSIE_REQUIRE(a.rstride >= cmax && a.partials != nullptr, VSIE_ERR_ARG, "seg_gemv: partial buffer");
  bool ok = false;
  switch (sl * 4 + mode) {
#define VSIE_SEGL(SL, M) \
  case SL * 4 + M: ok = launch_seg<M, SL>(a, ns, nq, smem, st); break;
    VSIE_SEGL(8, 1) VSIE_SEGL(8, 2) VSIE_SEGL(8, 3) VSIE_SEGL(12, 1) VSIE_SEGL(12, 2) VSIE_SEGL(12, 3)
    VSIE_SEGL(16, 1) VSIE_SEGL(16, 2) VSIE_SEGL(16, 3)
#undef VSIE_SEGL
    default: break;
  }
  if (!ok) return false;
  VSIE_CHECK_LAUNCH();
  if (mode & 2) {
    GemvN g{};
    g.nbatch = a.nbatch;
    for (int b = 0; b < a.nbatch; ++b) {
      g.y[b] = a.yt[b];
      g.R[b] = a.C[b];
    }
    launch_gemv_sum(g, a.partials, ns, a.rstride, st);
  }
  return true;
}

bool launch_seg_gemv(const SegGemv& a, bool transpose, cudaStream_t st) {
  return launch_seg_gemv_mode(a, transpose ? 2 : 1, st, false);
}

}  // namespace vsie
