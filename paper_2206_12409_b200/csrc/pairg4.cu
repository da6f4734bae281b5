// The G4 pass of one GMRES coupling matvec (SURVEY §8a A4 + A9), streamed by TMA.
//
// The forward's first step y4 = G4 x (Eq. 17) and the transpose's last step
// z = sum_chi (G4^chi)^T z3^chi (Eqs. 18-19) both read all of G4 (r3 x m,
// column-major, the largest core).  This kernel reads it ONCE for both, for up to the three
// chi components in one launch, and also forms the chi sum of Eq. 18 in fixed order.
//
// Per CTA: one contiguous column range [c0, c1) of every chi (the same range: every chi has
// m columns).  A producer warp streams that range, chi after chi, through a ring of 16
// shared-memory stages of <= 10 KB with 1-D bulk copies (cp.async.bulk, mbarrier
// complete_tx), so that ~160 KB per SM are in flight independent of how fast a column is
// retired.  Stage i is consumed by warp i % 8 alone (two stages per warp in flight, no
// cross-warp barrier per stage): lane l holds rows l + 32 q (q < NQ) of a column; columns
// are taken in pairs, the transpose dot products d = G4[:, c] . z3 of the pair are reduced
// by one half-exchange plus a 16-lane butterfly, the forward accumulation acc[q] +=
// G4[r, c] x[c] stays in registers until the chi is done, then a fixed-order smem tree over
// the warps gives the CTA's y4 partial (summed over CTAs by k_sum_partials_warp).  x and
// z3 are staged in shared memory once.  The z chi sum runs in a per-CTA smem accumulator,
// written once (conjugated for op C) after the last chi: deterministic, no atomics.
#include "common.cuh"
#include "kernels.cuh"
#include "tma_ring.cuh"

#include <cstdlib>

#include <algorithm>

namespace vsie {
namespace {
using namespace tma;

constexpr int kConsumerWarps = 8;
constexpr int kPairThreads = 32 * (kConsumerWarps + 1);   // + one producer warp
constexpr int kStageBytes = 10240;                       // >= 2 columns of r3 <= 320
constexpr int kRingMaxBytes = 16 * kStageBytes;          // 160 KB: two slots per consumer warp

// barrier over the 256 consumer threads only (the producer warp keeps streaming)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps) : "memory"); }

struct StageMap {
  int cps[3];      // columns per stage of chi b
  int nst[3];      // stages of chi b
  int off[3];      // first global stage of chi b
};

// Stage i (global over the chi sequence) lives in slot i % kSlots and is consumed by warp
// i % kConsumerWarps alone: no cross-warp barrier per stage, each warp double-buffered.
// MODE: 3 both products (the GMRES pair, G4-shared schedule), 1 forward only (y4 = G4 x),
// 2 transpose only (z = sum_chi G4^T z3) -- the single applies and the G3-shared pair
template <int NQ, int MODE, int SL>
__global__ void __launch_bounds__(kPairThreads, 1) k_pair_g4(const __grid_constant__ PairG4 a) {
  constexpr bool FW = (MODE & 1) != 0, TR = (MODE & 2) != 0;
  constexpr int kSlots = SL;                       // 16 slots: 160 KB in flight per SM
  constexpr int kRingBytes = SL * kStageBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  cplx* ring = reinterpret_cast<cplx*>(smem);
  cplx* red = reinterpret_cast<cplx*>(smem + kRingBytes);                 // [4][32 NQ]
  cplx* zacc = red + 4 * 32 * NQ;                                          // [c1 - c0]
  cplx* xs = zacc + a.ccta;                                                // x[c0 .. c1)
  cplx* zs = xs + a.ccta;                                                  // [3][32 NQ] z3
  __shared__ uint64_t full[kSlots], empty[kSlots];

  const int ns = gridDim.x, s = blockIdx.x;
  const int64_t C = a.C;
  const int64_t c0 = C * s / ns, c1 = C * (s + 1) / ns;
  const int nc = (int)(c1 - c0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StageMap mp;
  int total = 0;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    mp.cps[b] = 1;
    mp.nst[b] = 0;
    mp.off[b] = total;
    if (b < a.nbatch) {
      mp.cps[b] = max(1, kStageBytes / (int)(16 * a.R[b]));
      mp.nst[b] = (nc + mp.cps[b] - 1) / mp.cps[b];
      total += mp.nst[b];
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: G4 is constant and x is the caller's input, so the ring
    // is filled before waiting on the stream predecessor (programmatic dependent launch)
    if (lane == 0) {
      int i = 0;
      for (int b = 0; b < a.nbatch; ++b) {
        const int64_t R = a.R[b];
        for (int t = 0; t < mp.nst[b]; ++t, ++i) {
          const int slot = i % kSlots;
          if (i >= kSlots) mbar_wait(&empty[slot], ((i / kSlots) - 1) & 1);
          const int cb = t * mp.cps[b];
          const int ncol = min(mp.cps[b], nc - cb);
          const uint32_t bytes = (uint32_t)(16 * R * ncol);
          mbar_expect_tx(&full[slot], bytes);
          bulk_g2s(ring + (size_t)slot * (kStageBytes / 16), a.A[b] + R * (c0 + cb), bytes, &full[slot]);
        }
      }
    }
    pdl_wait();
    return;
  }

  // ---------------- consumers
  // x may be written by the caller's preceding kernel (the single forward apply starts with
  // this kernel): staged only after the PDL wait, from L2 (a per-column global load inside
  // the stage loop would sit behind the HBM stream's queues)
  pdl_wait();   // x / z3 come from the stream predecessor
  if (FW)
    for (int j = threadIdx.x; j < nc; j += 32 * kConsumerWarps) xs[j] = __ldcg(a.x + c0 + j);
  if (TR) {
    // all of a thread's z3 loads in flight before its stores (this sits after the PDL wait,
    // on the critical path)
    constexpr int PER = (3 * 32 * NQ + 32 * kConsumerWarps - 1) / (32 * kConsumerWarps);
    cplx v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + q * 32 * kConsumerWarps, b = e / (32 * NQ), r = e - b * 32 * NQ;
      v[q] = (b < a.nbatch && r < a.R[b]) ? __ldcg(a.z3[b] + r) : cmk(0, 0);   // rows past R: zero weight
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + q * 32 * kConsumerWarps;
      if (e < 3 * 32 * NQ) zs[e] = v[q];
    }
  }
  consumers_sync();
  for (int b = 0; b < a.nbatch; ++b) {
    const int R = (int)a.R[b];
    const int last = R - 1 - lane;
    const int cps = mp.cps[b];
    cplx zv[NQ], acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      zv[q] = TR ? zs[b * 32 * NQ + lane + 32 * q] : cmk(0, 0);
      acc[q] = cmk(0, 0);
    }
    // this warp's stages of chi b: global index i = off + t, t = warp - off mod 8, step 8
    const int off = mp.off[b];
    for (int t = (warp - off % kConsumerWarps + kConsumerWarps) % kConsumerWarps; t < mp.nst[b];
         t += kConsumerWarps) {
      const int i = off + t;
      const int slot = i % kSlots;
      const int cb = t * cps;
      const int ncol = min(cps, nc - cb);
      mbar_wait(&full[slot], (i / kSlots) & 1);
      const cplx* st = ring + (size_t)slot * (kStageBytes / 16);
      for (int j = 0; j < ncol; j += 2) {
        const bool two = j + 1 < ncol;
        const cplx* col = st + R * j;
        const cplx* col1 = two ? col + R : col;
        const cplx xv0 = FW ? xs[cb + j] : cmk(0, 0), xv1 = FW && two ? xs[cb + j + 1] : cmk(0, 0);
        cplx d0 = cmk(0, 0), d1 = cmk(0, 0);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int r = min(32 * q, last) + lane;   // rows past R re-read row R - 1 (zero weight)
          const cplx v0 = col[r], v1 = col1[r];
          if (TR) {
            cfma(d0, v0, zv[q]);
            cfma(d1, v1, zv[q]);
          }
          if (FW) {
            cfma(acc[q], v0, xv0);
            cfma(acc[q], v1, xv1);
          }
        }
        if (TR) {
          const cplx d = pair_reduce(d0, d1, lane);
          const int jj = cb + j + (lane >> 4);
          if ((lane & 15) == 0 && (lane == 0 || two)) zacc[jj] = b == 0 ? d : cadd(zacc[jj], d);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    // y4 partial of this CTA: fixed-order tree over the 8 warps (w += w + 4, w + 2, w + 1);
    // the barriers also order this chi's zacc updates before the next chi's
    if (!FW) {
      consumers_sync();   // orders this chi's zacc updates before the next chi's
      continue;
    }
#pragma unroll
    for (int half = kConsumerWarps / 2; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) red[(warp - half) * 32 * NQ + lane + 32 * q] = acc[q];
      }
      consumers_sync();
      if (warp < half) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = cadd(acc[q], red[warp * 32 * NQ + lane + 32 * q]);
      }
      consumers_sync();
    }
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = lane + 32 * q;
        if (r < R) {
          if (ns == 1)
            a.y4[b][r] = acc[q];
          else
            a.partials[((int64_t)b * ns + s) * a.rstride + r] = acc[q];
        }
      }
    }
  }
  pdl_trigger();
  if (TR)
    for (int j = threadIdx.x; j < nc; j += 32 * kConsumerWarps) {
      const cplx v = zacc[j];
      a.z[c0 + j] = a.conj_z ? cconj(v) : v;
    }
}


// ---------------------------------------------------------------- large r3 (320 < R <= 2048)
// Row-band variant for the r3 ~ 1500 cores of the two-surface configs (cfg 3 / 5): a lane
// can no longer hold a whole column, so every stage (whole columns, <= 32 KB) is consumed
// by ALL 8 consumer warps, warp w owning the row band [R w / 8, R (w + 1) / 8) (lane l:
// rows band0 + l + 32 q, q < NQ).  The forward accumulators of a band stay in that warp's
// registers (no cross-warp tree: the bands are disjoint); the transpose's per-column dot
// product is reduced across the lanes of each warp and kept as a per-(warp, column) partial
// in shared memory, summed over the chi (Eq. 18) and finally over the 8 warps in fixed
// order.  The stage's empty barrier counts the 8 warps.  Deterministic, no atomics.
constexpr int kBandMaxSlots = 16;

template <int NQ, int MODE>
__global__ void __launch_bounds__(kPairThreads, 1) k_pair_g4_band(const __grid_constant__ PairG4 a) {
  constexpr bool FW = (MODE & 1) != 0, TR = (MODE & 2) != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  const int nslots = a.nslots;
  const int64_t se = a.slot_elems;
  cplx* ring = reinterpret_cast<cplx*>(smem);
  cplx* zw = ring + (size_t)nslots * se;            // [8][ccta] per-warp column partials
  cplx* xs = zw + (size_t)kConsumerWarps * a.ccta;  // x[c0 .. c1)
  __shared__ uint64_t full[kBandMaxSlots], empty[kBandMaxSlots];

  const int ns = gridDim.x, s = blockIdx.x;
  const int64_t C = a.C;
  const int64_t c0 = C * s / ns, c1 = C * (s + 1) / ns;
  const int nc = (int)(c1 - c0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StageMap mp;
  int total = 0;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    mp.cps[b] = 1;
    mp.nst[b] = 0;
    mp.off[b] = total;
    if (b < a.nbatch) {
      mp.cps[b] = max(1, (int)(se / a.R[b]));
      mp.nst[b] = (nc + mp.cps[b] - 1) / mp.cps[b];
      total += mp.nst[b];
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // producer: G4 is constant -- the ring fills before the stream predecessor ends
    if (lane == 0) {
      int i = 0;
      for (int b = 0; b < a.nbatch; ++b) {
        const int64_t R = a.R[b];
        for (int t = 0; t < mp.nst[b]; ++t, ++i) {
          const int slot = i % nslots;
          if (i >= nslots) mbar_wait(&empty[slot], ((i / nslots) - 1) & 1);
          const int cb = t * mp.cps[b];
          const int ncol = min(mp.cps[b], nc - cb);
          const uint32_t bytes = (uint32_t)(16 * R * ncol);
          mbar_expect_tx(&full[slot], bytes);
          bulk_g2s(ring + (size_t)slot * se, a.A[b] + R * (c0 + cb), bytes, &full[slot]);
        }
      }
    }
    pdl_wait();
    return;
  }

  pdl_wait();   // x / z3 come from the stream predecessor
  if (FW)
    for (int j = threadIdx.x; j < nc; j += 32 * kConsumerWarps) xs[j] = __ldcg(a.x + c0 + j);
  consumers_sync();
  for (int b = 0; b < a.nbatch; ++b) {
    const int R = (int)a.R[b];
    const int rb0 = R * warp / kConsumerWarps, B = R * (warp + 1) / kConsumerWarps - rb0;
    const int last = B - 1 - lane;   // B >= 1 (R > 320)
    const int cps = mp.cps[b];
    cplx zv[NQ], acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      zv[q] = TR && lane + 32 * q < B ? __ldcg(a.z3[b] + rb0 + lane + 32 * q) : cmk(0, 0);   // past B: zero weight
      acc[q] = cmk(0, 0);
    }
    for (int t = 0; t < mp.nst[b]; ++t) {
      const int i = mp.off[b] + t;
      const int slot = i % nslots;
      const int cb = t * cps;
      const int ncol = min(cps, nc - cb);
      mbar_wait(&full[slot], (i / nslots) & 1);
      const cplx* st = ring + (size_t)slot * se + rb0;
      for (int j = 0; j < ncol; j += 2) {
        const bool two = j + 1 < ncol;
        const cplx* col = st + (int64_t)R * j;
        const cplx* col1 = two ? col + R : col;
        const cplx xv0 = FW ? xs[cb + j] : cmk(0, 0), xv1 = FW && two ? xs[cb + j + 1] : cmk(0, 0);
        cplx d0 = cmk(0, 0), d1 = cmk(0, 0);
        if (two) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int r = min(32 * q, last) + lane;   // rows past the band re-read its last row
            const cplx v0 = col[r], v1 = col1[r];
            if (TR) {
              cfma(d0, v0, zv[q]);
              cfma(d1, v1, zv[q]);
            }
            if (FW) {
              cfma(acc[q], v0, xv0);
              cfma(acc[q], v1, xv1);
            }
          }
        } else {   // a lone column (one column per stage at r3 ~ 1500): no duplicate reads
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const cplx v0 = col[min(32 * q, last) + lane];
            if (TR) cfma(d0, v0, zv[q]);
            if (FW) cfma(acc[q], v0, xv0);
          }
        }
        // the stage's last column pair is in registers: free the slot before the shuffle
        // reduction, so the refill does not wait on it (one column per stage at r3 ~ 1500)
        if (j + 2 >= ncol) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
        }
        if (TR) {
          const cplx d = pair_reduce(d0, d1, lane);
          const int jj = cb + j + (lane >> 4);
          cplx* zp = zw + (size_t)warp * a.ccta + jj;
          if ((lane & 15) == 0 && (lane == 0 || two)) *zp = b == 0 ? d : cadd(*zp, d);
        }
      }
    }
    if (FW) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int r = lane + 32 * q;
        if (r < B) {
          if (ns == 1)
            a.y4[b][rb0 + r] = acc[q];
          else
            a.partials[((int64_t)b * ns + s) * a.rstride + rb0 + r] = acc[q];
        }
      }
    }
  }
  pdl_trigger();
  if (TR) {
    consumers_sync();   // every warp's column partials complete
    for (int j = threadIdx.x; j < nc; j += 32 * kConsumerWarps) {
      cplx v = zw[j];
#pragma unroll
      for (int w = 1; w < kConsumerWarps; ++w) v = cadd(v, zw[(size_t)w * a.ccta + j]);
      a.z[c0 + j] = a.conj_z ? cconj(v) : v;
    }
  }
}

}  // namespace

int pair_g4_max_rank() { return 2048; }

namespace {

bool launch_pair_g4_band(const PairG4& a, int64_t rmax, int max_ctas, cudaStream_t st) {
  int64_t rmin = rmax;
  for (int b = 0; b < a.nbatch; ++b) rmin = std::min(rmin, a.R[b]);
  // the band kernel needs a non-empty band per warp: every chi's R > 8 (R > 320 for some chi;
  // a small R of another chi is handled too as long as it fills the 8 bands)
  if (rmin < kConsumerWarps) return false;
  const int nq = (int)ceil_div(ceil_div(rmax, kConsumerWarps), 32);
  const int ns = (int)std::max<int64_t>(1, std::min<int64_t>(max_ctas, ceil_div(a.C, 4)));
  const int64_t ccta = ceil_div(a.C, ns);
  // stage = whole columns, >= 16 KB; as many slots as fit beside the partials (<= 16)
  const int64_t se = std::max<int64_t>(rmax, 16384 / 16 / rmax * rmax);
  const size_t extra = (size_t)(kConsumerWarps + 1) * ccta * sizeof(cplx);
  // 170 KB rather than all of shared memory: cfg 3 pair 1.836 -> 1.808 ms (150 KB 1.816, 120 KB 1.829)
  const size_t budget = 170 * 1024;
  if (extra + 2 * se * sizeof(cplx) > budget) return false;
  const int nslots = (int)std::min<int64_t>(kBandMaxSlots, (budget - extra) / (se * sizeof(cplx)));
  const size_t smem = (size_t)nslots * se * sizeof(cplx) + extra;
  PairG4 b = a;
  b.ccta = ccta;
  b.nslots = nslots;
  b.slot_elems = se;
  const int mode = (a.x ? 1 : 0) | (a.z3[0] ? 2 : 0);
  if (mode == 0) return true;
  switch (nq * 4 + mode) {
#define VSIE_PGB(K, M)                                                                             \
  case K * 4 + M: {                                                                                \
    static size_t attr = 0;                                                                        \
    if (smem > attr) {                                                                             \
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_pair_g4_band<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      attr = smem;                                                                                 \
    }                                                                                              \
    launch_pdl(k_pair_g4_band<K, M>, dim3(ns), dim3(kPairThreads), smem, st, b);                   \
    break;                                                                                         \
  }
#define VSIE_PGB3(K) VSIE_PGB(K, 1) VSIE_PGB(K, 2) VSIE_PGB(K, 3)
    VSIE_PGB3(2) VSIE_PGB3(3) VSIE_PGB3(4) VSIE_PGB3(5) VSIE_PGB3(6) VSIE_PGB3(7) VSIE_PGB3(8)
#undef VSIE_PGB3
#undef VSIE_PGB
    default: return false;
  }
  VSIE_CHECK_LAUNCH();
  if (ns > 1 && a.x) {
    GemvN g{};
    g.nbatch = a.nbatch;
    for (int q = 0; q < a.nbatch; ++q) {
      g.y[q] = a.y4[q];
      g.R[q] = a.R[q];
    }
    launch_gemv_sum(g, a.partials, ns, a.rstride, st);
  }
  return true;
}

}  // namespace

bool launch_pair_g4(const PairG4& a, int max_ctas, cudaStream_t st) {
  int64_t rmax = 0;
  for (int b = 0; b < a.nbatch; ++b) rmax = std::max(rmax, a.R[b]);
  if (rmax > 2048 || rmax < 1) return false;
  if (a.C == 0) return true;
  VSIE_REQUIRE(a.rstride >= rmax, VSIE_ERR_ARG, "pair_g4: partial stride below r3");
  if (rmax > 320) return launch_pair_g4_band(a, rmax, max_ctas, st);
  const int nq = (int)ceil_div(rmax, 32);
  const int ns = (int)std::max<int64_t>(1, std::min<int64_t>(max_ctas, ceil_div(a.C, 4)));
  const int64_t ccta = ceil_div(a.C, ns);
  const size_t smem = kRingMaxBytes + (size_t)4 * 32 * nq * sizeof(cplx) + (size_t)2 * ccta * sizeof(cplx) +
                      (size_t)3 * 32 * nq * sizeof(cplx);
  PairG4 b = a;
  b.ccta = ccta;
  if (smem > 220 * 1024) return false;
  const int mode = (a.x ? 1 : 0) | (a.z3[0] ? 2 : 0);
  if (mode == 0) return true;
  switch (nq * 4 + mode) {
#define VSIE_PG4M(K, M)                                                                            \
  case K * 4 + M: {                                                                                \
    static size_t attr = 0;                                                                        \
    if (smem > attr) {                                                                             \
      VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_pair_g4<K, M, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
      attr = smem;                                                                                 \
    }                                                                                              \
    launch_pdl(k_pair_g4<K, M, 16>, dim3(ns), dim3(kPairThreads), smem, st, b);                    \
    break;                                                                                         \
  }
#define VSIE_PG4(K) VSIE_PG4M(K, 1) VSIE_PG4M(K, 2) VSIE_PG4M(K, 3)
    VSIE_PG4(1) VSIE_PG4(2) VSIE_PG4(3) VSIE_PG4(4) VSIE_PG4(5) VSIE_PG4(6) VSIE_PG4(7) VSIE_PG4(8) VSIE_PG4(9)
    VSIE_PG4(10)
#undef VSIE_PG4
#undef VSIE_PG4M
    default: return false;
  }
  VSIE_CHECK_LAUNCH();
  if (ns > 1 && a.x) {
    GemvN g{};
    g.nbatch = a.nbatch;
    for (int b = 0; b < a.nbatch; ++b) {
      g.y[b] = a.y4[b];
      g.R[b] = a.R[b];
    }
    launch_gemv_sum(g, a.partials, ns, a.rstride, st);
  }
  return true;
}

}  // namespace vsie
