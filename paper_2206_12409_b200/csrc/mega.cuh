// Persistent dataflow apply ("megakernel") for single right-hand sides.
//
// One launch per apply direction runs every TT-contraction step of all three chi
// components (Eq. 17 forward, Eqs. 18-19 transpose) as a queue of tiles that
// the resident CTAs claim in order through an atomic counter.  A tile waits (spins on
// an acquire flag) only for the tiles it reads from; those were claimed earlier, so the
// queue cannot deadlock, and the steps of different chi overlap instead of being
// separated by kernel boundaries (ramp / tail / launch gaps of ~3 us per kernel on
// B200, measured in tools/microbench/stream_gemv.cu).  All split reductions are done by
// the last-arriving tile of a group in a fixed order: results are bitwise reproducible.
//
// Forward steps (queue phases):  0 y4 = G4 x        (split columns, ticket-reduced)
//                                1 Y3 = G3 y4       (row blocks)
//                                2 Y2 = G2 Y3       (DMMA GEMM tiles)
//                                3 y  = G1 Y2       (DMMA expansion tiles, voxel writes)
// Transpose steps:               0 W1 = G1^T u      (DMMA reduction tiles, voxel reads)
//                                1 W2 = G2^T W1     (DMMA GEMM tiles, split-K ticket-reduced)
//                                2 z3 = G3^T W2     (row ranges x column chunks, ticket-reduced)
//                                3 z  = sum_chi G4^T z3   (column chunks, chi sum by ticket)
#pragma once

#include "kernels.cuh"

#include <vector>

namespace vsie {

constexpr int kMegaPhases = 4;

struct MegaChi {
  const cplx* G1;   // n1 x r1
  const cplx* G2;   // (r1 n2) x r2
  const cplx* G3;   // (r2 n3l) x r3: the shard's i3 slice
  const cplx* G4;   // r3 x mloc: the shard's columns
  int r1, r2, r3;
};

// Tile plan (host-computed by mega_plan; per chi where ranks differ)
struct MegaPlan {
  // forward
  int nrb4[3], s4[3];      // phase 0: row blocks (<= 128 rows) x column splits
  int nrb3[3], s3[3];      // phase 1: row ranges (<= 256 rows) over the r2 n3l rows of G3 x column splits
  int gm_f[3], gn_f;       // forward GEMM tiles (64 x 32): m blocks per chi, n blocks of 32 planes
  int gm_a[3], gn_a;       // transpose GEMM tiles (32 x 64): m blocks per chi, n blocks of 64 planes
  int gs[3];               // transpose GEMM split-K
  int ecols, ne;           // expansion / reduction tiles: columns per tile, tiles per chi
  // transpose
  int nrr3[3], ncc3[3];    // phase 2: row ranges x 32-column chunks
  int cc4, ncc4;           // phase 3: columns per chunk, chunks
  // queue: segments of (phase, chi) in claim order; every (phase, chi) segment comes
  // after (phase - 1, chi), which is all the dependency order the tiles need
  int nseg;
  int seg_phase[12], seg_chi[12], seg_off[13];
  int count[kMegaPhases][3];   // tiles of (phase, chi)
  // sync words (offsets into MegaArgs::sync)
  int o_tick_a[3], o_cnt_a[3], o_flag_a[3];   // fwd: y4 tickets per row block / cnt / ready
  int o_flag_b[3], o_tick_b[3];              // fwd: Y3 row range ready / split tickets
  int o_cnt_c[3], o_flag_c[3];               // fwd: Y2 n-block counters / ready;  adj: W2 n-block
  int o_flag_e[3];                           // adj: W1 reduction tile ready
  int o_tick_g[3];                           // adj: split-K tickets per GEMM tile
  int o_tick_z[3], o_cnt_z[3], o_flag_z[3];  // adj: z3 tickets per column chunk / cnt / ready
  int o_tick_s;                              // adj: chi-sum tickets per G4 chunk
  int sync_words;
  int grid_fwd, grid_adj;    // resident CTAs (occupancy x SMs) of the two kernels
  int smem_fwd, smem_adj;    // dynamic shared memory bytes
  // partial buffers (complex elements)
  int64_t p_a[3], p_b[3], p_g[3], p_z[3], p_s;
  int64_t part_elems;
};

struct MegaArgs {
  MegaChi c[3];
  int n1, n2, n3l;
  int64_t mloc;
  int r3max, r2max, r1max;
  MegaPlan p;
  // io (single RHS): forward x = the shard's surface columns, y = voxel vector (chi
  // blocks chi_stride apart, this shard's planes at vox_off); transpose x = voxel vector,
  // y = the shard's surface columns
  const cplx* x;
  cplx* y;
  int64_t chi_stride, vox_off;
  int conj;
  // workspaces
  cplx* y4;        // [3][r3max]          forward y4 / transpose z3 (reduced)
  cplx* Y3;        // [3][r2max n3l]      forward Y3 / transpose W2
  cplx* Y2;        // [3][r1max n2 n3l]   forward Y2 / transpose W1
  cplx* zpart;     // [3][mloc]           transpose per-chi G4^T z3
  cplx* part;      // partial sums (plan offsets)
  unsigned* sync;  // [0] tile counter, [1] done counter, [2] epoch, then plan words (zeroed once)
  int phase_begin, phase_end;  // queue phases run by this launch (world > 1 splits at the collective)
  unsigned long long* trace;   // diagnostics (null = off): per tile {t0 ns, t1 ns, smid, ready ns}
};

// diagnostics: per-tile timeline of the last traced launch of a direction
struct MegaTraceRec {
  int phase, chi;
  int64_t idx;
  int sm;
  double t0_us, t1_us, tr_us;   // claimed, finished, dependencies satisfied
};

// host side
void mega_plan(MegaArgs& a);
// launches; when a.trace is set, *plan_out receives the plan with the claim order used
void launch_mega(const MegaArgs& a, bool forward, cudaStream_t st, MegaPlan* plan_out = nullptr);
// decodes a trace buffer (count = plan.seg_off[plan.nseg] tiles) into records
std::vector<MegaTraceRec> mega_decode_trace(const MegaPlan& plan, const unsigned long long* host_trace);

}  // namespace vsie
