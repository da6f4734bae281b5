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

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kCW) : "memory"); }

// M: 1 op N (x -> y), 2 op T (xt -> yt through partials), 3 both from ONE pass over the core.
// The ring has a.nslots stages of a.stage_elems (whole column segments of the CTA's row
// block, ~12 KB) chosen by the launcher to fill the shared memory left beside the vectors
// (<= 16 slots; a chain's per-chi pass uses a small ring so that the neighbouring chain's
// compute kernels fit beside it on the SMs).
constexpr int kMaxSlots = 16;

template <int NQ, int M>
__global__ void __launch_bounds__(kSegThreads, 1) k_seg_gemv(const __grid_constant__ SegGemv a) {
  constexpr bool FW = (M & 1) != 0, OPT = (M & 2) != 0;
  const int kSlotsS = a.nslots;
  const int64_t se = a.stage_elems;
  extern __shared__ __align__(128) unsigned char smem[];
  cplx* ring = reinterpret_cast<cplx*>(smem);
  // [max(Cmax, 4 * 32 NQ)]: the op T partial z (vec) and the op N warp tree (red) share it
  // (the partial is written out, behind a barrier, before the tree of the same chi)
  cplx* vec = ring + (size_t)kSlotsS * se;
  cplx* red = vec;
  cplx* vecx = vec + (OPT ? max(a.cmax, (int64_t)(FW ? 4 * 32 * NQ : 0)) : 4 * 32 * NQ);   // [Cmax]: x (op N)
  __shared__ uint64_t full[kMaxSlots], empty[kMaxSlots];
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
      seg[b] = L[b] > 0 ? max(1, (int)(se / L[b])) : 1;   // column segments per stage
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
          bulk_g2s(ring + (size_t)slot * se, a.A[b] + a.C[b] * r0[b] + (int64_t)L[b] * cb, sb * ncol,
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
        const cplx* st = ring + (size_t)slot * se;
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

template <int M>
bool launch_seg(const SegGemv& a, int ns, int nq, size_t smem, cudaStream_t st) {
  switch (nq) {
#define VSIE_SEG(K)                                                                                  \
  case K: {                                                                                          \
    static size_t attr = 0;                                                                          \
    if (smem > attr) {                                                                               \
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_seg_gemv<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      attr = smem;                                                                                   \
    }                                                                                                \
    launch_pdl(k_seg_gemv<K, M>, dim3(ns), dim3(kSegThreads), smem, st, a);                          \
    return true;                                                                                     \
  }
    VSIE_SEG(1) VSIE_SEG(2) VSIE_SEG(3) VSIE_SEG(4) VSIE_SEG(5) VSIE_SEG(6) VSIE_SEG(7) VSIE_SEG(8)
    VSIE_SEG(10) VSIE_SEG(12) VSIE_SEG(16)
#undef VSIE_SEG
    default: return false;
  }
}

// ring geometry of a launch: stages of whole column segments (~12 KB), as many slots (<= 16)
// as fit beside the vectors (op T partial / op N tree, aliased, + op N x); the chains' per-chi
// passes take an 80 KB ring.  false if not even two slots fit.
bool seg_geometry(int64_t L, int nq, int64_t cmax, int mode, bool small_ring, int* nslots, int64_t* se,
                  size_t* smem) {
  const bool fw = mode & 1, opt = mode & 2;
  const int64_t vec = opt ? std::max<int64_t>(cmax, fw ? 4 * 32 * nq : 0) : 4 * 32 * nq;
  const size_t extra = (size_t)(vec + (fw ? cmax : 0)) * sizeof(cplx);
  if (extra >= 220 * 1024) return false;
  const size_t budget = small_ring ? 80 * 1024 : 220 * 1024 - extra;
  // stage i is consumed by warp i % kCW alone, so the slot count is a multiple of kCW (8 or
  // 16): every slot is then always consumed by the same warp, in order, and no warp can wait
  // on a slot phase ahead of one another warp has not consumed.  Stages of whole segments,
  // <= 24 KB; the slot count with more bytes in flight wins (16 on a tie).
  int64_t n = 0, segb = 0;
  for (int cand : {16, 8}) {
    const int64_t sg = std::min<int64_t>((int64_t)(budget / (cand * 16 * L)), std::max<int64_t>(1, 24576 / (16 * L)));
    if (sg >= 1 && cand * sg > n * segb) {
      n = cand;
      segb = sg;
    }
  }
  if (n == 0) return false;
  *se = segb * L;
  *nslots = (int)n;
  *smem = (size_t)n * *se * sizeof(cplx) + extra;
  return *smem <= 220 * 1024;
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
  if (L > 512) return false;
  int ns;
  int64_t se;
  size_t smem;
  return seg_geometry(L, seg_nq(L), C, 3, false, &ns, &se, &smem);
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
  if (L > 512) return false;
  const int nq = seg_nq(L);
  a.cmax = cmax;
  size_t smem = 0;
  if (!seg_geometry(L, nq, cmax, mode, small_ring, &a.nslots, &a.stage_elems, &smem)) return false;
  if (mode & 2) VSIE_REQUIRE(a.rstride >= cmax && a.partials != nullptr, VSIE_ERR_ARG, "seg_gemv: partial buffer");
  const bool ok = mode == 1 ? launch_seg<1>(a, ns, nq, smem, st)
                  : mode == 2 ? launch_seg<2>(a, ns, nq, smem, st)
                              : launch_seg<3>(a, ns, nq, smem, st);
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
