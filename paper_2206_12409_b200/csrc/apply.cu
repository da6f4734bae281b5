// The TT apply of Z_bc: forward y = Z x (Eq. 17) and plain /
// conjugate transpose z = Z^T u, Z^H u (Eqs. 18-19), orchestrated over the
// kernels of ttapply.cu / linalg.cu.
//
// Each chi component is an independent TT, so an apply is three independent
// kernel chains (SURVEY §8d "chi-pipelining"): chain chi runs on its own stream,
//   forward   : y4 = G4 x -> Y3 = G3 y4 -> Y2 = G2 Y3 -> y_chi = G1 Y2
//   transpose : W1 = G1^T u_chi -> W2 = G2^T W1 -> z3 = G3^T W2 -> z_chi = G4^T z3
// and the transpose's Eq. 18 sum over chi is one small deterministic kernel at the join.
// The three chains overlap one another's launch gaps, ramp-up and tails.  The whole
// fork/join DAG is captured once per (op, nrhs, x, y) as a CUDA graph and replayed on the
// caller's stream (no host launch overhead per kernel).  With the slab partition
// (SURVEY §8e design iii) the chains join around the cross-rank combines of y4 / z3.
#include <algorithm>
#include <cstdlib>

#include "handle.hpp"

namespace vsie {

// ------------------------------------------------------------------ per-kernel timing scopes
struct Scope {
  vsie_coupling_s* h;
  size_t slot = 0;
  bool on;
  cudaStream_t stream = nullptr;
  unsigned flags = cudaEventRecordDefault;   // external event nodes inside captures
  Scope(vsie_coupling_s* hh, const char* name, int64_t bytes, int64_t flops, cudaStream_t st) : h(hh), on(hh->timing) {
    if (!on) return;
    Timed t;
    t.name = name;
    t.bytes = bytes;
    t.flops = flops;
    VSIE_REQUIRE(h->event_pool.size() >= 2, VSIE_ERR_STATE,
                 "timing event pool exhausted: read the timers (vsie_coupling_timers / _trace) more often");
    t.e0 = h->event_pool.back();
    h->event_pool.pop_back();
    t.e1 = h->event_pool.back();
    h->event_pool.pop_back();
    t.chi = h->scope_chi;
    t.call = h->trace_call;
    t.origin = h->trace_origin;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    VSIE_CHECK_CUDA(cudaStreamIsCapturing(st, &cs));
    flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    VSIE_CHECK_CUDA(cudaEventRecordWithFlags(t.e0, st, flags));
    h->pending.push_back(t);
    slot = h->pending.size() - 1;
    stream = st;
  }
  ~Scope() {
    if (on) cudaEventRecordWithFlags(h->pending[slot].e1, stream, flags);
  }
};

namespace {

// copy a (rows x cols) column-major block with source ld / dest ld
void copy2d(cplx* dst, int64_t ldd, const cplx* src, int64_t lds, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  VSIE_CHECK_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(cplx), src, lds * sizeof(cplx), rows * sizeof(cplx), cols,
                                    cudaMemcpyDeviceToDevice, st));
}

struct IoLayout {
  int64_t chi_stride;  // elements between chi blocks of the voxel-side vector
  int64_t ld;          // elements between RHS columns
  bool global;         // buffer is the global 3 n_v vector (world 1 / loopback)
};

IoLayout voxel_layout(vsie_coupling_s* h) {
  IoLayout L;
  const int64_t n12 = (int64_t)h->grid.n[0] * h->grid.n[1];
  if (h->comm) {
    const int64_t local = n12 * h->shards[0].n3loc();
    L.chi_stride = local;
    L.ld = 3 * local;
    L.global = false;
  } else {
    L.chi_stride = h->grid.nv();
    L.ld = 3 * h->grid.nv();
    L.global = true;
  }
  return L;
}

int64_t shard_voxel_offset(vsie_coupling_s* h, const Shard& s, const IoLayout& L) {
  return L.global ? (int64_t)h->grid.n[0] * h->grid.n[1] * s.i3b : 0;
}

struct Ctx {
  vsie_coupling_s* h;
  int k;            // nrhs
  int r1m, r2m, r3m;
  int64_t r3stride;  // r3m * k
  IoLayout L;
  int ws = 0;       // 0: forward workspaces, 3: the transpose's (both directions concurrently)
  cplx* partials(int c) const { return h->partials.p + (c + ws) * h->partials_per_chi; }
  cplx* zws(int c) const { return h->zgemm_ws.p + (c + ws) * h->zgemm_ws_per_chi; }
  int64_t R(int c, int j) const { return h->ranks[c][j]; }
};

constexpr int kMaxSplits = 256;

// GMRES pair schedule: 0 = k_gemv_nt per chi chain, 2 = one TMA-streamed launch over the
// three chi (k_pair_g4, chi sum of Eq. 18 fused), 3 = forward and transpose as six
// independent concurrent chains (single shard only), 4 = every step one batched launch,
// 5 = streaming passes overlapped with the other direction's G1 / G2 chains (G4 read
// twice, G3 once for both directions; single shard); VSIE_PAIR_G4 overrides
int pair_g4_mode() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_PAIR_G4");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}

// the GMRES pair's G4 pass per chi inside the chains (small ring), followed there by that
// chi's G3 / G2 / G1 steps; VSIE_G4_CHAIN=1
bool g4_chain_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_G4_CHAIN");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// the transpose's G1^T, G2^T and G3^T per chi inside the chains (small-ring k_seg_gemv);
// VSIE_ADJ_CHAIN_SEG=1
bool adj_chain_seg_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_ADJ_CHAIN_SEG");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// the forward's G3 pass per chi inside the chains (small-ring k_seg_gemv) instead of one
// batched pass before them, so one chi's G2 / G1 work runs beside the next chi's G3 stream.
// Measured: cfg 2 (34 MB of G3 per chi) 0.1606 -> 0.1565 ms; cfg 4 (64 MB per chi) 0.4553 ->
// 0.4594 ms.  Default: on when the largest per-chi G3 slice is <= 48 MB;
// VSIE_FWD_CHAIN_SEG=1 / 0 forces it on / off.
bool fwd_chain_seg_on(const vsie_coupling_s* h) {
  static const int v = [] {
    const char* e = std::getenv("VSIE_FWD_CHAIN_SEG");
    return e ? std::atoi(e) : -1;
  }();
  if (v >= 0) return v != 0;
  int64_t mx = 0;
  for (const Shard& s : h->shards)
    for (int c = 0; c < 3; ++c) mx = std::max<int64_t>(mx, 16LL * h->ranks[c][1] * s.n3loc() * h->ranks[c][2]);
  return mx <= (48LL << 20);
}

// batched TMA-streamed G3 steps in the pair (k_seg_gemv); VSIE_SEG_G3=0 keeps the per-chi GEMVs
bool seg_g3_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_SEG_G3");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// leave the G2^T split-K partials for the batched G3^T kernel to sum on load instead of a
// split-K reduce launch: measured slower (cfg 2 pair 0.165 -> 0.171 ms: the partial loads
// sit at the head of every CTA) -- opt-in, VSIE_W2_PARTS=1
bool w2_parts_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_W2_PARTS");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// fused transpose front (k_adj12: G1^T and G2^T in one launch over the three chi) in the
// pair, opt-in VSIE_ADJ_FUSED=1: measured slower (cfg 2 pair 0.167 -> 0.195 ms): the G2
// slices of the three resident CTAs per SM (3 x 91 KB) do not stay in L1 (65% hit rate)
// and the lanes-over-beta contraction waits on L2
bool adj_fused_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_ADJ_FUSED");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

bool fuse_g21() {
  // fused G2 + G1 forward tail (k_g21_fwd): measured 0.173 vs 0.167 ms per pair step at
  // cfg 2 (its 110 KB of smem leave one CTA per SM) -- opt-in
  static const int v = [] {
    const char* e = std::getenv("VSIE_FUSE_G21");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// ------------------------------------------------------------------ forward chain pieces (one chi)
// step 1: y4 = G4[:, owned] x[owned], partial per shard
void fwd_g4(const Ctx& X, Shard& s, int c, const cplx* x, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  cplx* y4 = s.y4.p + c * X.r3stride;
  if (s.mloc() == 0) {
    VSIE_CHECK_CUDA(cudaMemsetAsync(y4, 0, X.r3stride * sizeof(cplx), st));
    return;
  }
  if (k == 1) {
    GemvN g{};
    g.nbatch = 1;
    g.A[0] = s.G4[c].p;
    g.x[0] = x + s.cb;
    g.y[0] = y4;
    g.R[0] = X.R(c, 2);
    g.C[0] = s.mloc();
    const int64_t bytes = 16 * (X.R(c, 2) * s.mloc() + s.mloc() + X.R(c, 2));
    Scope sc(h, "fwd_g4_gemv", bytes, 8 * X.R(c, 2) * s.mloc(), st);
    launch_gemv_n(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
  } else {
    Zgemm z{};
    z.nbatch = 1;
    z.M[0] = X.R(c, 2); z.N[0] = k; z.K[0] = s.mloc();
    z.A[0] = s.G4[c].p; z.lda[0] = X.R(c, 2);
    z.B[0] = x + s.cb; z.ldb[0] = h->m;
    z.C[0] = y4; z.ldc[0] = X.R(c, 2);
    const int64_t bytes = 16 * (X.R(c, 2) * s.mloc() + (s.mloc() + X.R(c, 2)) * k);
    Scope sc(h, "fwd_g4_zgemm", bytes, 8 * X.R(c, 2) * s.mloc() * k, st);
    launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
  }
}

// steps 2-4 on the owned planes: Y3 = G3 y4, Y2 = G2 Y3, y = G1 Y2
void fwd_rest(const Ctx& X, Shard& s, int c, cplx* y, cudaStream_t st, cudaEvent_t mid = nullptr, bool with_g3 = true) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  if (n3l == 0) return;
  const int64_t r1 = X.R(c, 0), r2 = X.R(c, 1), r3 = X.R(c, 2);
  cplx* y4 = s.y4.p + c * X.r3stride;
  cplx* Y3 = s.Y3.p + c * X.r2m * n3l * k;
  cplx* Y2 = s.Y2.p + c * X.r1m * n2 * n3l * k;
  if (!with_g3) {
    // Y3 already formed (batched k_seg_gemv)
  } else if (k == 1) {
    GemvN g{};
    g.nbatch = 1;
    g.A[0] = s.G3[c].p;
    g.x[0] = y4;
    g.y[0] = Y3;
    g.R[0] = r2 * n3l;
    g.C[0] = r3;
    const int64_t bytes = 16 * (r2 * n3l * r3 + r2 * n3l + r3);
    Scope sc(h, "fwd_g3_gemv", bytes, 8 * r2 * n3l * r3, st);
    launch_gemv_n(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
  } else {
    Zgemm z{};
    z.nbatch = 1;
    z.M[0] = r2 * n3l; z.N[0] = k; z.K[0] = r3;
    z.A[0] = s.G3[c].p; z.lda[0] = r2 * n3l;
    z.B[0] = y4; z.ldb[0] = r3;
    z.C[0] = Y3; z.ldc[0] = r2 * n3l;
    const int64_t bytes = 16 * (r2 * n3l * r3 + (r2 * n3l + r3) * k);
    Scope sc(h, "fwd_g3_zgemm", bytes, 8 * r2 * n3l * r3 * k, st);
    launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
  }
  if (mid) VSIE_CHECK_CUDA(cudaEventRecord(mid, st));   // chain staggering: G3 stream done
  if (k == 1 && fuse_g21()) {
    // Y2 = G2 Y3 and y = G1 Y2 in one kernel (Y2 tiles stay in shared memory)
    G21Args f{};
    f.G1 = h->G1[c].p;
    f.G2 = h->G2[c].p;
    f.Y3 = Y3;
    f.y = y + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    f.n1 = n1;
    f.n2 = n2;
    f.n3l = (int)n3l;
    f.r1 = (int)r1;
    f.r2 = (int)r2;
    bool done;
    {
      const int64_t bytes = 16 * ((int64_t)n1 * r1 + r1 * n2 * r2 + r2 * n3l + (int64_t)n1 * n2 * n3l);
      Scope sc(h, "fwd_g21_fused", bytes, 8 * (r1 * n2 * r2 * n3l + (int64_t)n1 * r1 * n2 * n3l), st);
      done = launch_g21_fwd(f, st);
    }
    if (done) return;
  }
  {
    Zgemm z{};
    z.nbatch = 1;
    z.M[0] = r1 * n2; z.N[0] = n3l * k; z.K[0] = r2;
    z.A[0] = h->G2[c].p; z.lda[0] = r1 * n2;
    z.B[0] = Y3; z.ldb[0] = r2;
    z.C[0] = Y2; z.ldc[0] = r1 * n2;
    const int64_t bytes = 16 * (r1 * n2 * r2 + r2 * n3l * k + r1 * n2 * n3l * k);
    Scope sc(h, "fwd_g2_zgemm", bytes, 8 * r1 * n2 * r2 * n3l * k, st);
    launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
  }
  {
    ExpandArgs e{};
    e.nbatch = 1;
    e.n1 = n1;
    e.ncol = (int64_t)n2 * n3l * k;
    e.cols_per_rhs = (int64_t)n2 * n3l;
    e.ld_rhs = X.L.ld;
    e.G1[0] = h->G1[c].p;
    e.Y2[0] = Y2;
    e.y[0] = y + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    e.r1[0] = (int)r1;
    const int64_t bytes = 16 * ((int64_t)n1 * r1 + r1 * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k);
    Scope sc(h, "fwd_g1_expand", bytes, 8 * (int64_t)n1 * r1 * n2 * n3l * k, st);
    launch_expand_g1(e, st);
  }
}

// ------------------------------------------------------------------ transpose chain pieces (one chi)
// W1 = G1^T u, W2 = G2^T W1, z3 = G3^T W2: partial z3 per shard
void adj_front(const Ctx& X, Shard& s, int c, const cplx* u, bool cj, cudaStream_t st, cudaEvent_t mid = nullptr,
               bool with_g3 = true, bool with_g1 = true, bool with_g2 = true) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  cplx* z3 = s.z3.p + c * X.r3stride;
  if (n3l == 0) {
    VSIE_CHECK_CUDA(cudaMemsetAsync(z3, 0, X.r3stride * sizeof(cplx), st));
    return;
  }
  const int64_t r1 = X.R(c, 0), r2 = X.R(c, 1), r3 = X.R(c, 2);
  cplx* W1 = s.W1.p + c * X.r1m * n2 * n3l * k;
  cplx* W2 = s.W2.p + c * X.r2m * n3l * k;
  if (!with_g2) {
    // G2^T by the batched k_g2t after the chains (only G1^T here)
    ReduceArgs r{};
    r.nbatch = 1;
    r.n1 = n1;
    r.ncol = (int64_t)n2 * n3l * k;
    r.cols_per_rhs = (int64_t)n2 * n3l;
    r.ld_rhs = X.L.ld;
    r.conj_u = cj;
    r.G1[0] = h->G1[c].p;
    r.u[0] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    r.W1[0] = W1;
    r.r1[0] = (int)r1;
    const int64_t bytes = 16 * ((int64_t)n1 * r1 + r1 * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k);
    Scope sc(h, "adj_g1_reduce", bytes, 8 * (int64_t)n1 * r1 * n2 * n3l * k, st);
    launch_reduce_g1(r, st);
    return;
  }
  if (with_g1) {
    ReduceArgs r{};
    r.nbatch = 1;
    r.n1 = n1;
    r.ncol = (int64_t)n2 * n3l * k;
    r.cols_per_rhs = (int64_t)n2 * n3l;
    r.ld_rhs = X.L.ld;
    r.conj_u = cj;
    r.G1[0] = h->G1[c].p;
    r.u[0] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    r.W1[0] = W1;
    r.r1[0] = (int)r1;
    const int64_t bytes = 16 * ((int64_t)n1 * r1 + r1 * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k);
    Scope sc(h, "adj_g1_reduce", bytes, 8 * (int64_t)n1 * r1 * n2 * n3l * k, st);
    launch_reduce_g1(r, st);
  }
  {
    Zgemm z{};
    z.nbatch = 1;
    z.ta = kT;
    z.M[0] = r2; z.N[0] = n3l * k; z.K[0] = r1 * n2;
    z.A[0] = h->G2[c].p; z.lda[0] = r1 * n2;
    z.B[0] = W1; z.ldb[0] = r1 * n2;
    z.C[0] = W2; z.ldc[0] = r2;
    const int64_t bytes = 16 * (r1 * n2 * r2 + r2 * n3l * k + r1 * n2 * n3l * k);
    h->w2_parts[c] = 0;
    int parts = 0;
    int64_t stride = 0;
    {
      // the GEMM and its split-K sum are timed as two kernels (bench roofline per kernel)
      Scope sc(h, "adj_g2_zgemm", bytes, 8 * r1 * n2 * r2 * n3l * k, st);
      parts = launch_zgemm_dmma_parts(z, X.zws(c), h->zgemm_ws_per_chi, st, &stride);
    }
    if (parts > 0) {
      if (!with_g3 && k == 1 && h->shards.size() == 1 && w2_parts_on()) {
        // the batched G3^T kernel sums the split-K partials of W2 on load
        h->w2_parts[c] = parts;
        h->w2_part_stride[c] = stride;
      } else {
        Scope sc(h, "adj_g2_splitk_sum", 16 * (parts + 1) * r2 * n3l * k, 8 * parts * r2 * n3l * k, st);
        launch_splitk_sum(z, X.zws(c), parts, stride, st);
      }
    }
  }
  if (mid) VSIE_CHECK_CUDA(cudaEventRecord(mid, st));   // chain staggering: G1/G2 steps done
  if (!with_g3) return;   // z3 by the batched k_seg_gemv
  if (k == 1) {
    GemvT g{};
    g.nbatch = 1;
    g.A[0] = s.G3[c].p;
    g.x[0] = W2;
    g.y[0] = z3;
    g.R[0] = r2 * n3l;
    g.C[0] = r3;
    const int64_t bytes = 16 * (r2 * n3l * r3 + r2 * n3l + r3);
    Scope sc(h, "adj_g3_gemv", bytes, 8 * r2 * n3l * r3, st);
    launch_gemv_t(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
  } else {
    Zgemm z{};
    z.nbatch = 1;
    z.ta = kT;
    z.M[0] = r3; z.N[0] = k; z.K[0] = r2 * n3l;
    z.A[0] = s.G3[c].p; z.lda[0] = r2 * n3l;
    z.B[0] = W2; z.ldb[0] = r2 * n3l;
    z.C[0] = z3; z.ldc[0] = r3;
    const int64_t bytes = 16 * (r2 * n3l * r3 + (r2 * n3l + r3) * k);
    Scope sc(h, "adj_g3_zgemm", bytes, 8 * r2 * n3l * r3 * k, st);
    launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
  }
}

// z_chi[owned] = G4[:, owned]^T z3 into the shard's per-chi partial
void adj_g4(const Ctx& X, Shard& s, int c, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int64_t ml = s.mloc();
  if (ml == 0) return;
  const int64_t r3 = X.R(c, 2);
  const int64_t ldz = s.zpart.n / (3 * k);
  cplx* zp = s.zpart.p + c * ldz * k;
  const cplx* z3 = s.z3.p + c * X.r3stride;
  if (k == 1) {
    GemvT g{};
    g.nbatch = 1;
    g.A[0] = s.G4[c].p;
    g.x[0] = z3;
    g.y[0] = zp;
    g.R[0] = r3;
    g.C[0] = ml;
    const int64_t bytes = 16 * (r3 * ml + r3 + ml);
    Scope sc(h, "adj_g4_gemv", bytes, 8 * r3 * ml, st);
    launch_gemv_t(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
  } else {
    Zgemm z{};
    z.nbatch = 1;
    z.ta = kT;
    z.M[0] = ml; z.N[0] = k; z.K[0] = r3;
    z.A[0] = s.G4[c].p; z.lda[0] = r3;
    z.B[0] = z3; z.ldb[0] = r3;
    z.C[0] = zp; z.ldc[0] = ldz;
    const int64_t bytes = 16 * (r3 * ml + (r3 + ml) * k);
    Scope sc(h, "adj_g4_zgemm", bytes, 8 * r3 * ml * k, st);
    launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
  }
}

// Eq. 18: z[owned] = sum_chi z_chi (fixed order), conj for op C
void adj_sum_chi(const Ctx& X, Shard& s, cplx* zout, int64_t ldz_out, bool cj, cudaStream_t st) {
  const int64_t ml = s.mloc();
  if (ml == 0) return;
  const int64_t ldz = s.zpart.n / (3 * X.k);
  Scope sc(X.h, "adj_sum_chi", 16 * 4 * ml * X.k, 0, st);
  launch_sum3(s.zpart.p, ldz * X.k, ldz, ml, X.k, zout, ldz_out, cj, st);
}

// sum the per-shard partial vectors (3 r3max nrhs) across ranks / shards
void combine_r3(vsie_coupling_s* h, DevBuf<cplx> Shard::*buf, int64_t n, cudaStream_t st) {
  if (h->comm) {
    Scope sc(h, "nccl_allreduce", 0, 0, st);
    h->comm->allreduce_sum(reinterpret_cast<double*>((h->shards[0].*buf).p), 2 * (size_t)n, st);
    return;
  }
  if (h->shards.size() <= 1) return;
  Scope sc(h, "loopback_allreduce", 0, 0, st);
  cplx* acc = (h->shards[0].*buf).p;
  for (size_t s = 1; s < h->shards.size(); ++s) launch_axpy1((h->shards[s].*buf).p, acc, n, st);
  for (size_t s = 1; s < h->shards.size(); ++s)
    VSIE_CHECK_CUDA(cudaMemcpyAsync((h->shards[s].*buf).p, acc, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
}

bool stagger_on() {
  // measured at cfg 2: staggered chains 0.29 ms vs 0.20 ms concurrent -- off by default
  static const int v = [] {
    const char* e = std::getenv("VSIE_STAGGER");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// ------------------------------------------------------------------ fork / join
void ensure_streams(vsie_coupling_s* h) {
  if (h->chi_stream[0]) return;
  // chain chi gets stream priority rank chi (0 highest): the block scheduler then runs
  // chain 0 at full width and lets chains 1, 2 fill its ramp / tail / dependency bubbles
  int least = 0, greatest = 0;
  VSIE_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  static const int prio_on = [] {
    const char* e = std::getenv("VSIE_CHAIN_PRIORITY");
    return e ? std::atoi(e) : 1;
  }();
  for (int c = 0; c < 3; ++c) {
    int prio = greatest + c;
    if (prio > least) prio = least;
    if (!prio_on) prio = least;
    VSIE_CHECK_CUDA(cudaStreamCreateWithPriority(&h->chi_stream[c], cudaStreamNonBlocking, prio));
    VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_join[c], cudaEventDisableTiming));
    VSIE_CHECK_CUDA(cudaStreamCreateWithPriority(&h->chi_stream2[c], cudaStreamNonBlocking, prio));
    VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_join2[c], cudaEventDisableTiming));
  }
  VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  for (int c = 0; c < 3; ++c) VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_stage[c], cudaEventDisableTiming));
  VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
}

struct Streams {
  cudaStream_t main;
  cudaStream_t chi[3];
  bool parallel;
  cudaStream_t chi2[3];   // second chain set (set only where a DAG uses it)
};

Streams make_streams(vsie_coupling_s* h, cudaStream_t main, bool parallel) {
  if (!parallel) return Streams{main, {main, main, main}, false, {main, main, main}};
  return Streams{main, {h->chi_stream[0], h->chi_stream[1], h->chi_stream[2]}, true,
                 {h->chi_stream2[0], h->chi_stream2[1], h->chi_stream2[2]}};
}

void fork(vsie_coupling_s* h, const Streams& S, bool both = false) {
  if (!S.parallel) return;
  VSIE_CHECK_CUDA(cudaEventRecord(h->ev_fork, S.main));
  for (int c = 0; c < 3; ++c) VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.chi[c], h->ev_fork, 0));
  if (both)
    for (int c = 0; c < 3; ++c) VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.chi2[c], h->ev_fork, 0));
}

void join(vsie_coupling_s* h, const Streams& S, bool both = false) {
  if (!S.parallel) return;
  for (int c = 0; c < 3; ++c) {
    VSIE_CHECK_CUDA(cudaEventRecord(h->ev_join[c], S.chi[c]));
    VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.main, h->ev_join[c], 0));
  }
  if (both)
    for (int c = 0; c < 3; ++c) {
      VSIE_CHECK_CUDA(cudaEventRecord(h->ev_join2[c], S.chi2[c]));
      VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.main, h->ev_join2[c], 0));
    }
}

// ------------------------------------------------------------------ persistent single-RHS apply
bool mega_ready(vsie_coupling_s* h) {
  static const int env = [] {
    const char* e = std::getenv("VSIE_MEGA");
    return e ? std::atoi(e) : 1;
  }();
  if (!env || h->apply_mode != 1) return false;
  for (const Shard& s : h->shards)
    if (!s.mega.sync) return false;
  return true;
}

// algorithmic bytes of one direction on one shard
int64_t mega_bytes(vsie_coupling_s* h, const Shard& s) {
  int64_t b = 16 * (s.mloc() + 3 * (int64_t)h->grid.n[0] * h->grid.n[1] * s.n3loc());
  for (int c = 0; c < 3; ++c) {
    const int64_t r1 = h->ranks[c][0], r2 = h->ranks[c][1], r3 = h->ranks[c][2];
    b += 16 * (h->grid.n[0] * r1 + r1 * h->grid.n[1] * r2 + r2 * s.n3loc() * r3 + r3 * s.mloc());
  }
  return b;
}

void mega_launch(vsie_coupling_s* h, Shard& s, const cplx* x, cplx* y, bool fwd, int conj, int pb, int pe,
                 const IoLayout& L, cudaStream_t st) {
  MegaArgs a = s.mega;
  a.x = fwd ? x + s.cb : x;
  a.y = y;
  a.chi_stride = L.chi_stride;
  a.vox_off = shard_voxel_offset(h, s, L);
  a.conj = conj;
  a.phase_begin = pb;
  a.phase_end = pe;
  const bool whole = pb == 0 && pe == kMegaPhases;
  Scope sc(h, fwd ? (whole ? "fwd_mega" : "fwd_mega_part") : (whole ? "adj_mega" : "adj_mega_part"),
           whole ? mega_bytes(h, s) : 0, 0, st);
  if (h->tile_trace) {
    const int d = fwd ? 0 : 1;
    VSIE_REQUIRE(s.mega_trace[d].p != nullptr, VSIE_ERR_STATE, "tile trace buffers not allocated");
    VSIE_CHECK_CUDA(cudaMemsetAsync(s.mega_trace[d].p, 0, s.mega_trace[d].bytes(), st));
    a.trace = s.mega_trace[d].p;
    launch_mega(a, fwd, st, &s.mega_traced[d]);
    return;
  }
  launch_mega(a, fwd, st);
}

void apply_mega(vsie_coupling_s* h, const cplx* x, cplx* y, int op, cudaStream_t st) {
  const IoLayout L = voxel_layout(h);
  const bool exchange = h->comm != nullptr || h->shards.size() > 1;
  int r3m = 1;
  for (int c = 0; c < 3; ++c) r3m = std::max(r3m, h->ranks[c][2]);
  static const int dbg_pe = [] {   // diagnostics: run only phases [0, VSIE_MEGA_PHASE_END)
    const char* e = std::getenv("VSIE_MEGA_PHASE_END");
    return e ? std::atoi(e) : kMegaPhases;
  }();
  if (op == VSIE_OP_N) {
    if (!exchange) {
      mega_launch(h, h->shards[0], x, y, true, 0, 0, dbg_pe, L, st);
      return;
    }
    for (Shard& s : h->shards) mega_launch(h, s, x, y, true, 0, 0, 1, L, st);
    combine_r3(h, &Shard::y4, 3 * (int64_t)r3m, st);   // allreduce of y4
    for (Shard& s : h->shards) mega_launch(h, s, x, y, true, 0, 1, kMegaPhases, L, st);
    return;
  }
  const int cj = op == VSIE_OP_C;
  const int64_t m = h->m, mp = ceil_div(m, h->world);
  auto out_of = [&](Shard& s) -> cplx* {
    return h->comm ? h->gather_buf.p + (int64_t)h->world * mp : y + s.cb;
  };
  if (!exchange) {
    mega_launch(h, h->shards[0], x, out_of(h->shards[0]), false, cj, 0, dbg_pe, L, st);
    return;
  }
  for (Shard& s : h->shards) mega_launch(h, s, x, out_of(s), false, cj, 0, kMegaPhases - 1, L, st);
  combine_r3(h, &Shard::y4, 3 * (int64_t)r3m, st);     // allreduce of z3
  for (Shard& s : h->shards) mega_launch(h, s, x, out_of(s), false, cj, kMegaPhases - 1, kMegaPhases, L, st);
  if (h->comm) {
    Scope sc(h, "nccl_allgather", 0, 0, st);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) VSIE_CHECK_CUDA(cudaMemsetAsync(seg + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), st));
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p), 2 * (size_t)mp,
                       st);
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(y + cb, m, h->gather_buf.p + (int64_t)p * mp, mp, ce - cb, 1, st);
    }
  }
}

// ------------------------------------------------------------------ batched single-stream apply
// One launch per contraction step covering all three chi (nbatch = 3): fewer, larger
// kernels than the per-chi chains (each kernel's launch / ramp / tail is paid once per
// step for the three components), in the order of Eq. 17 / Eqs. 18-19; the transpose's
// last GEMV sums over chi inside the kernel (Eq. 18).
void apply_batched(vsie_coupling_s* h, const cplx* x, cplx* y, int op, cudaStream_t st) {
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t m = h->m;
  int r1m = 1, r2m = 1, r3m = 1;
  for (int c = 0; c < 3; ++c) {
    r1m = std::max(r1m, h->ranks[c][0]);
    r2m = std::max(r2m, h->ranks[c][1]);
    r3m = std::max(r3m, h->ranks[c][2]);
  }
  const IoLayout L = voxel_layout(h);
  auto R = [&](int c, int j) { return (int64_t)h->ranks[c][j]; };
  const bool exchange = h->comm != nullptr || h->shards.size() > 1;
  cplx* part = h->partials.p;
  const int64_t pcap = 3 * h->partials_per_chi;
  cplx* zws = h->zgemm_ws.p;
  const int64_t zcap = 3 * h->zgemm_ws_per_chi;
  if (op == VSIE_OP_N) {
    for (Shard& s : h->shards) {
      if (s.mloc() == 0) {
        VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p, 0, s.y4.bytes(), st));
        continue;
      }
      GemvN g{};
      g.nbatch = 3;
      int64_t bytes = 16 * s.mloc(), fl = 0;
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G4[c].p;
        g.x[c] = x + s.cb;
        g.y[c] = s.y4.p + c * r3m;
        g.R[c] = R(c, 2);
        g.C[c] = s.mloc();
        bytes += 16 * (R(c, 2) * s.mloc() + R(c, 2));
        fl += 8 * R(c, 2) * s.mloc();
      }
      Scope sc(h, "fwd_g4_gemv", bytes, fl, st);
      launch_gemv_n(g, part, pcap, kMaxSplits, st);
    }
    if (exchange) combine_r3(h, &Shard::y4, 3 * (int64_t)r3m, st);
    for (Shard& s : h->shards) {
      const int64_t n3l = s.n3loc();
      if (n3l == 0) continue;
      {
        GemvN g{};
        g.nbatch = 3;
        int64_t bytes = 0, fl = 0;
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G3[c].p;
          g.x[c] = s.y4.p + c * r3m;
          g.y[c] = s.Y3.p + c * r2m * n3l;
          g.R[c] = R(c, 1) * n3l;
          g.C[c] = R(c, 2);
          bytes += 16 * (R(c, 1) * n3l * R(c, 2) + R(c, 1) * n3l + R(c, 2));
          fl += 8 * R(c, 1) * n3l * R(c, 2);
        }
        Scope sc(h, "fwd_g3_gemv", bytes, fl, st);
        launch_gemv_n(g, part, pcap, kMaxSplits, st);
      }
      {
        Zgemm z{};
        z.nbatch = 3;
        int64_t bytes = 0, fl = 0;
        for (int c = 0; c < 3; ++c) {
          z.M[c] = R(c, 0) * n2; z.N[c] = n3l; z.K[c] = R(c, 1);
          z.A[c] = h->G2[c].p; z.lda[c] = R(c, 0) * n2;
          z.B[c] = s.Y3.p + c * r2m * n3l; z.ldb[c] = R(c, 1);
          z.C[c] = s.Y2.p + c * r1m * n2 * n3l; z.ldc[c] = R(c, 0) * n2;
          bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l + R(c, 0) * n2 * n3l);
          fl += 8 * R(c, 0) * n2 * R(c, 1) * n3l;
        }
        Scope sc(h, "fwd_g2_zgemm", bytes, fl, st);
        launch_zgemm_dmma(z, zws, zcap, st);
      }
      {
        ExpandArgs e{};
        e.nbatch = 3;
        e.n1 = n1;
        e.ncol = (int64_t)n2 * n3l;
        e.cols_per_rhs = e.ncol;
        e.ld_rhs = L.ld;
        int64_t bytes = 0, fl = 0;
        for (int c = 0; c < 3; ++c) {
          e.G1[c] = h->G1[c].p;
          e.Y2[c] = s.Y2.p + c * r1m * n2 * n3l;
          e.y[c] = y + c * L.chi_stride + shard_voxel_offset(h, s, L);
          e.r1[c] = (int)R(c, 0);
          bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l + (int64_t)n1 * n2 * n3l);
          fl += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l;
        }
        Scope sc(h, "fwd_g1_expand", bytes, fl, st);
        launch_expand_g1(e, st);
      }
    }
    return;
  }
  const bool cj = op == VSIE_OP_C;
  for (Shard& s : h->shards) {
    const int64_t n3l = s.n3loc();
    if (n3l == 0) {
      VSIE_CHECK_CUDA(cudaMemsetAsync(s.z3.p, 0, s.z3.bytes(), st));
      continue;
    }
    {
      ReduceArgs r{};
      r.nbatch = 3;
      r.n1 = n1;
      r.ncol = (int64_t)n2 * n3l;
      r.cols_per_rhs = r.ncol;
      r.ld_rhs = L.ld;
      r.conj_u = cj;
      int64_t bytes = 0, fl = 0;
      for (int c = 0; c < 3; ++c) {
        r.G1[c] = h->G1[c].p;
        r.u[c] = x + c * L.chi_stride + shard_voxel_offset(h, s, L);
        r.W1[c] = s.Y2.p + c * r1m * n2 * n3l;
        r.r1[c] = (int)R(c, 0);
        bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l + (int64_t)n1 * n2 * n3l);
        fl += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l;
      }
      Scope sc(h, "adj_g1_reduce", bytes, fl, st);
      launch_reduce_g1(r, st);
    }
    {
      Zgemm z{};
      z.nbatch = 3;
      z.ta = kT;
      int64_t bytes = 0, fl = 0;
      for (int c = 0; c < 3; ++c) {
        z.M[c] = R(c, 1); z.N[c] = n3l; z.K[c] = R(c, 0) * n2;
        z.A[c] = h->G2[c].p; z.lda[c] = R(c, 0) * n2;
        z.B[c] = s.Y2.p + c * r1m * n2 * n3l; z.ldb[c] = R(c, 0) * n2;
        z.C[c] = s.W2.p + c * r2m * n3l; z.ldc[c] = R(c, 1);
        bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l + R(c, 0) * n2 * n3l);
        fl += 8 * R(c, 0) * n2 * R(c, 1) * n3l;
      }
      Scope sc(h, "adj_g2_zgemm", bytes, fl, st);
      launch_zgemm_dmma(z, zws, zcap, st);
    }
    {
      GemvT g{};
      g.nbatch = 3;
      int64_t bytes = 0, fl = 0;
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G3[c].p;
        g.x[c] = s.W2.p + c * r2m * n3l;
        g.y[c] = s.z3.p + c * r3m;
        g.R[c] = R(c, 1) * n3l;
        g.C[c] = R(c, 2);
        bytes += 16 * (R(c, 1) * n3l * R(c, 2) + R(c, 1) * n3l + R(c, 2));
        fl += 8 * R(c, 1) * n3l * R(c, 2);
      }
      Scope sc(h, "adj_g3_gemv", bytes, fl, st);
      launch_gemv_t(g, part, pcap, kMaxSplits, st);
    }
  }
  if (exchange) combine_r3(h, &Shard::z3, 3 * (int64_t)r3m, st);
  const int64_t mp = ceil_div(m, h->world);
  for (Shard& s : h->shards) {
    if (s.mloc() == 0) continue;
    GemvT g{};
    g.nbatch = 3;
    g.sum_batch = true;
    g.conj_out = cj;
    int64_t bytes = 16 * s.mloc(), fl = 0;
    cplx* zout = h->comm ? h->gather_buf.p + (int64_t)h->world * mp : y + s.cb;
    for (int c = 0; c < 3; ++c) {
      g.A[c] = s.G4[c].p;
      g.x[c] = s.z3.p + c * r3m;
      g.y[c] = zout;
      g.R[c] = R(c, 2);
      g.C[c] = s.mloc();
      bytes += 16 * (R(c, 2) * s.mloc() + R(c, 2));
      fl += 8 * R(c, 2) * s.mloc();
    }
    Scope sc(h, "adj_g4_gemv", bytes, fl, st);
    launch_gemv_t(g, part, pcap, kMaxSplits, st);
  }
  if (h->comm) {
    Scope sc(h, "nccl_allgather", 0, 0, st);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) VSIE_CHECK_CUDA(cudaMemsetAsync(seg + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), st));
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p), 2 * (size_t)mp,
                       st);
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(y + cb, m, h->gather_buf.p + (int64_t)p * mp, mp, ce - cb, 1, st);
    }
  }
}

// ------------------------------------------------------------------ the apply DAG
// forward G2 step for the three chi as one k_g2n launch (pair and single applies), opt-in
// VSIE_G2N=1: measured slower than the per-chi ZGEMM chains (cfg 2 pair 0.160 -> 0.166 ms:
// one warp per 8 x 8 tile re-reads G2 from L2 for every n-tile)
bool g2n_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_G2N");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

void launch_g2n_shard(vsie_coupling_s* h, const Ctx& X, Shard& s, cudaStream_t st) {
  const int n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  if (n3l == 0) return;
  G2tArgs g{};
  g.nbatch = 3;
  g.N = (int)n3l;
  int64_t bytes = 0, fl = 0;
  for (int c = 0; c < 3; ++c) {
    g.G2[c] = h->G2[c].p;
    g.W1[c] = s.Y3.p + c * X.r2m * n3l;
    g.W2[c] = s.Y2.p + c * X.r1m * n2 * n3l;
    g.M[c] = (int)(X.R(c, 0) * n2);
    g.K[c] = (int)X.R(c, 1);
    g.ldw[c] = (int)(X.R(c, 0) * n2);
    bytes += 16 * (X.R(c, 0) * n2 * X.R(c, 1) + X.R(c, 1) * n3l + X.R(c, 0) * n2 * n3l);
    fl += 8 * X.R(c, 0) * n2 * X.R(c, 1) * n3l;
  }
  Scope sc(h, "fwd_g2_g2n", bytes, fl, st);
  launch_g2n(g, st);
}

// the G1 expansion of one chi (Y2 formed)
void fwd_expand(const Ctx& X, Shard& s, int c, cplx* y, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  if (n3l == 0) return;
  const int64_t r1 = X.R(c, 0);
  ExpandArgs e{};
  e.nbatch = 1;
  e.n1 = n1;
  e.ncol = (int64_t)n2 * n3l;
  e.cols_per_rhs = e.ncol;
  e.ld_rhs = X.L.ld;
  e.G1[0] = h->G1[c].p;
  e.Y2[0] = s.Y2.p + c * X.r1m * n2 * n3l;
  e.y[0] = y + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
  e.r1[0] = (int)r1;
  const int64_t bytes = 16 * ((int64_t)n1 * r1 + r1 * n2 * n3l + (int64_t)n1 * n2 * n3l);
  Scope sc(h, "fwd_g1_expand", bytes, 8 * (int64_t)n1 * r1 * n2 * n3l, st);
  launch_expand_g1(e, st);
}

// batched W2 = G2^T W1 (k_g2t) instead of the per-chi split-K ZGEMM chains; VSIE_G2T=0
bool g2t_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_G2T");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// k_g2t per chi inside the chains (right after that chi's G1^T) instead of one batched
// launch after the join; VSIE_G2T_CHAIN=1
bool g2t_chain_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_G2T_CHAIN");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

// chi_only >= 0: the single chi chi_only (nbatch 1), else the three chi in one launch
void launch_g2t_shard(vsie_coupling_s* h, const Ctx& X, Shard& s, cudaStream_t st, int chi_only = -1) {
  const int n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  if (n3l == 0) return;
  G2tArgs g{};
  g.nbatch = chi_only >= 0 ? 1 : 3;
  g.N = (int)n3l;
  int64_t bytes = 0, fl = 0;
  for (int i = 0; i < g.nbatch; ++i) {
    const int c = chi_only >= 0 ? chi_only : i;
    g.G2[i] = h->G2[c].p;
    g.W1[i] = s.W1.p + c * X.r1m * n2 * n3l;
    g.W2[i] = s.W2.p + c * X.r2m * n3l;
    g.M[i] = (int)X.R(c, 1);
    g.K[i] = (int)(X.R(c, 0) * n2);
    g.ldw[i] = (int)X.R(c, 1);
    h->w2_parts[c] = 0;
    bytes += 16 * (X.R(c, 0) * n2 * X.R(c, 1) + X.R(c, 1) * n3l + X.R(c, 0) * n2 * n3l);
    fl += 8 * X.R(c, 0) * n2 * X.R(c, 1) * n3l;
  }
  Scope sc(h, "adj_g2_g2t", bytes, fl, st);
  launch_g2t(g, st);
}

// single applies (one RHS) on the batched TMA passes: forward = ONE G4 pass (y4, three chi)
// -> ONE G3 pass (Y3) -> per-chi G2 / G1 chains; transpose = G1^T (one TMA launch when it
// fits, else in the chains) -> per-chi G2^T chains -> ONE G3^T pass -> ONE G4^T pass with
// the Eq. 18 chi sum.  VSIE_SINGLE_TMA=0 keeps the per-chi chains of k_gemv_n / k_gemv_t.
bool single_tma_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_SINGLE_TMA");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

bool tma_shapes_ok(vsie_coupling_s* h, const Ctx& X) {
  if (X.r3m > pair_g4_max_rank()) return false;
  for (Shard& s : h->shards) {
    if (s.n3loc() == 0 || s.mloc() == 0) return false;
    for (int c = 0; c < 3; ++c)
      if (!seg_gemv_supported(X.R(c, 1) * s.n3loc(), X.R(c, 2), s.g3b_ns)) return false;
  }
  return true;
}

void apply_single_tma(vsie_coupling_s* h, Ctx X, const cplx* x, cplx* y, int op, const Streams& S) {
  const bool exchange = h->comm != nullptr || h->shards.size() > 1;
  const int64_t m = h->m, mp = ceil_div(m, h->world);
  const int64_t rsum = X.R(0, 2) + X.R(1, 2) + X.R(2, 2);
  if (op == VSIE_OP_N) {
    for (Shard& s : h->shards) {
      PairG4 p{};
      p.nbatch = 3;
      p.C = s.mloc();
      p.x = x + s.cb;
      p.partials = X.partials(0);
      p.rstride = X.r3m;
      for (int c = 0; c < 3; ++c) {
        p.A[c] = s.G4[c].p;
        p.y4[c] = s.y4.p + c * X.r3stride;
        p.R[c] = X.R(c, 2);
      }
      Scope sc(h, "fwd_g4_tma", 16 * rsum * (p.C + 1) + 16 * p.C, 8 * rsum * p.C, S.main);
      VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), S.main), VSIE_ERR_STATE, "single apply: G4 shape");
    }
    if (exchange) combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
    const bool chain_seg = fwd_chain_seg_on(h) && !g2n_on();   // as in the pair (pair_dag)
    for (Shard& s : h->shards) {
      if (chain_seg) break;
      const int64_t n3l = s.n3loc();
      SegGemv g{};
      g.nbatch = 3;
      g.nsb = s.g3b_ns;
      int64_t bytes = 0;
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G3b[c].p;
        g.x[c] = s.y4.p + c * X.r3stride;
        g.y[c] = s.Y3.p + c * X.r2m * n3l;
        g.R[c] = X.R(c, 1) * n3l;
        g.C[c] = X.R(c, 2);
        bytes += 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]);
      }
      Scope sc(h, "fwd_g3_seg", bytes, bytes / 2, S.main);
      VSIE_REQUIRE(launch_seg_gemv(g, false, S.main), VSIE_ERR_STATE, "single apply: G3 shape");
    }
    if (g2n_on())
      for (Shard& s : h->shards) launch_g2n_shard(h, X, s, S.main);
    fork(h, S);
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) {
        if (chain_seg) {
          const int64_t n3l = s.n3loc();
          SegGemv g{};
          g.nbatch = 1;
          g.nsb = s.g3b_ns;
          g.A[0] = s.G3b[c].p;
          g.x[0] = s.y4.p + c * X.r3stride;
          g.y[0] = s.Y3.p + c * X.r2m * n3l;
          g.R[0] = X.R(c, 1) * n3l;
          g.C[0] = X.R(c, 2);
          const int64_t bytes = 16 * (g.R[0] * g.C[0] + g.R[0] + g.C[0]);
          Scope sc(h, "fwd_g3_seg_chi", bytes, bytes / 2, S.chi[c]);
          VSIE_REQUIRE(launch_seg_gemv_mode(g, 1, S.chi[c], true), VSIE_ERR_STATE, "single apply: G3 shape");
        }
        if (g2n_on())
          fwd_expand(X, s, c, y, S.chi[c]);
        else
          fwd_rest(X, s, c, y, S.chi[c], nullptr, false);
      }
    }
    h->scope_chi = -1;
    join(h, S);
    return;
  }
  const bool cj = op == VSIE_OP_C;
  X.ws = 3;   // the transpose's own workspaces: a forward apply may run beside it
  bool g1_done = false;
  if (reduce_tma_on() && reduce_tma_fits(h->grid.n[0], X.r1m)) {
    g1_done = true;
    for (Shard& s : h->shards) {
      const int64_t n3l = s.n3loc();
      ReduceArgs r{};
      r.nbatch = 3;
      r.n1 = h->grid.n[0];
      r.ncol = (int64_t)h->grid.n[1] * n3l;
      r.cols_per_rhs = r.ncol;
      r.ld_rhs = X.L.ld;
      r.conj_u = cj;
      int64_t bytes = 0, fl = 0;
      for (int c = 0; c < 3; ++c) {
        r.G1[c] = h->G1[c].p;
        r.u[c] = x + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
        r.W1[c] = s.W1.p + c * X.r1m * h->grid.n[1] * n3l;
        r.r1[c] = (int)X.R(c, 0);
        bytes += 16 * ((int64_t)r.n1 * X.R(c, 0) + X.R(c, 0) * r.ncol + (int64_t)r.n1 * r.ncol);
        fl += 8 * (int64_t)r.n1 * X.R(c, 0) * r.ncol;
      }
      Scope sc(h, "adj_g1_reduce_tma", bytes, fl, S.main);
      VSIE_REQUIRE(launch_reduce_g1_tma(r, S.main), VSIE_ERR_STATE, "single apply: G1 shape");
    }
  }
  const bool g2b = g2t_on();
  if (!(g1_done && g2b)) {
    fork(h, S);
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) adj_front(X, s, c, x, cj, S.chi[c], nullptr, false, !g1_done, !g2b);
    }
    h->scope_chi = -1;
    join(h, S);
  }
  if (g2b)
    for (Shard& s : h->shards) launch_g2t_shard(h, X, s, S.main);
  for (Shard& s : h->shards) {
    const int64_t n3l = s.n3loc();
    SegGemv g{};
    g.nbatch = 3;
    g.nsb = s.g3b_ns;
    g.partials = X.partials(0);
    g.rstride = X.r3m;
    int64_t bytes = 0;
    for (int c = 0; c < 3; ++c) {
      g.A[c] = s.G3b[c].p;
      g.x[c] = s.W2.p + c * X.r2m * n3l;
      g.xparts[c] = 0;
      g.y[c] = s.z3.p + c * X.r3stride;
      g.R[c] = X.R(c, 1) * n3l;
      g.C[c] = X.R(c, 2);
      bytes += 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]);
    }
    Scope sc(h, "adj_g3_seg", bytes, bytes / 2, S.main);
    VSIE_REQUIRE(launch_seg_gemv(g, true, S.main), VSIE_ERR_STATE, "single apply: G3 shape");
  }
  if (exchange) combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
  for (Shard& s : h->shards) {
    PairG4 p{};
    p.nbatch = 3;
    p.C = s.mloc();
    p.z = h->comm ? h->gather_buf.p + (int64_t)h->world * mp : y + s.cb;
    p.conj_z = cj;
    p.partials = X.partials(0);
    p.rstride = X.r3m;
    for (int c = 0; c < 3; ++c) {
      p.A[c] = s.G4[c].p;
      p.z3[c] = s.z3.p + c * X.r3stride;
      p.R[c] = X.R(c, 2);
    }
    Scope sc(h, "adj_g4_tma", 16 * rsum * (p.C + 1) + 16 * p.C, 8 * rsum * p.C, S.main);
    VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), S.main), VSIE_ERR_STATE, "single apply: G4 shape");
  }
  if (h->comm) {
    Scope sc(h, "nccl_allgather", 0, 0, S.main);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) VSIE_CHECK_CUDA(cudaMemsetAsync(seg + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), S.main));
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p), 2 * (size_t)mp,
                       S.main);
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(y + cb, m, h->gather_buf.p + (int64_t)p * mp, mp, ce - cb, 1, S.main);
    }
  }
}

void apply_dag(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, const Streams& S) {
  if (nrhs == 1 && mega_ready(h)) {
    apply_mega(h, x, y, op, S.main);
    return;
  }
  if (nrhs == 1 && h->apply_mode == 2) {
    apply_batched(h, x, y, op, S.main);
    return;
  }
  Ctx X;
  X.h = h;
  X.k = nrhs;
  X.r1m = X.r2m = X.r3m = 1;
  for (int c = 0; c < 3; ++c) {
    X.r1m = std::max(X.r1m, h->ranks[c][0]);
    X.r2m = std::max(X.r2m, h->ranks[c][1]);
    X.r3m = std::max(X.r3m, h->ranks[c][2]);
  }
  X.r3stride = (int64_t)X.r3m * nrhs;
  X.L = voxel_layout(h);
  const bool exchange = h->comm != nullptr || h->shards.size() > 1;
  if (nrhs == 1 && single_tma_on() && tma_shapes_ok(h, X)) {
    apply_single_tma(h, X, x, y, op, S);
    return;
  }
  fork(h, S);
  if (op == VSIE_OP_N) {
    if (!exchange && stagger_on() && S.parallel) {
      // staggered chains: chain c+1 starts streaming G4 when chain c has finished its G3
      // stream, so one chain's tensor-core G2 / G1 steps overlap the next chain's HBM streams
      for (int c = 0; c < 3; ++c) {
        h->scope_chi = c;
        if (c > 0) VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.chi[c], h->ev_stage[c - 1], 0));
        fwd_g4(X, h->shards[0], c, x, S.chi[c]);
        fwd_rest(X, h->shards[0], c, y, S.chi[c], h->ev_stage[c]);
      }
      h->scope_chi = -1;
      join(h, S);
      return;
    }
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) fwd_g4(X, s, c, x, S.chi[c]);
    }
    h->scope_chi = -1;
    if (exchange) {
      // allreduce of the partial y4 (3 r3 values per RHS)
      join(h, S);
      combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
      fork(h, S);
    }
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) fwd_rest(X, s, c, y, S.chi[c]);
    }
    h->scope_chi = -1;
    join(h, S);
    return;
  }
  const bool cj = op == VSIE_OP_C;
  const bool stag = !exchange && stagger_on() && S.parallel;
  X.ws = 3;   // the transpose's own workspaces: a forward apply may run beside it
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    if (stag && c > 0) VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.chi[c], h->ev_stage[c - 1], 0));
    for (Shard& s : h->shards) adj_front(X, s, c, x, cj, S.chi[c], stag ? h->ev_stage[c] : nullptr);
  }
  h->scope_chi = -1;
  if (exchange) {
    join(h, S);
    combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
    fork(h, S);
  }
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) adj_g4(X, s, c, S.chi[c]);
  }
  h->scope_chi = -1;
  join(h, S);
  const int64_t m = h->m;
  const int64_t mp = ceil_div(m, h->world);
  const int k = nrhs;
  for (Shard& s : h->shards) {
    if (h->comm) {
      cplx* seg = h->gather_buf.p + (int64_t)h->world * mp * k;  // local segment staging [mp x k]
      adj_sum_chi(X, s, seg, mp, cj, S.main);
    } else {
      adj_sum_chi(X, s, y + s.cb, m, cj, S.main);
    }
  }
  if (h->comm) {
    // allgather of the column segments -> replicated z
    Scope sc(h, "nccl_allgather", 0, 0, S.main);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp * k;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) {
      for (int j = 0; j < k; ++j)
        VSIE_CHECK_CUDA(cudaMemsetAsync(seg + mp * j + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), S.main));
    }
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p),
                       2 * (size_t)mp * k, S.main);
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(y + cb, m, h->gather_buf.p + (int64_t)p * mp * k, mp, ce - cb, k, S.main);
    }
  }
}

bool graphs_enabled(vsie_coupling_s* h) {
  static const int env = [] {
    const char* e = std::getenv("VSIE_APPLY_GRAPHS");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0) return false;
  if (!h->use_graphs || h->timing || h->tile_trace) return false;
  // NCCL collectives inside captured graphs are not exercised on this pool's
  // 1-GPU boxes: the multi-rank path runs the same DAG eagerly unless forced on.
  if (h->comm && env != 1) return false;
  return true;
}

}  // namespace

void apply_reset_graphs(vsie_coupling_s* h) {
  for (GraphEntry& g : h->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  h->graphs.clear();
}

void apply_destroy(vsie_coupling_s* h) {
  apply_reset_graphs(h);
  for (int c = 0; c < 3; ++c) {
    if (h->chi_stream[c]) cudaStreamDestroy(h->chi_stream[c]);
    if (h->ev_join[c]) cudaEventDestroy(h->ev_join[c]);
    if (h->chi_stream2[c]) cudaStreamDestroy(h->chi_stream2[c]);
    if (h->ev_join2[c]) cudaEventDestroy(h->ev_join2[c]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  for (int c = 0; c < 3; ++c)
    if (h->ev_stage[c]) cudaEventDestroy(h->ev_stage[c]);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
}

namespace {

// Runs an apply DAG under the current timing / graph policy.  `dag(S)` enqueues the
// work on the Streams it is given; graphs are cached by (op, nrhs, x, y, u, z).
template <class Dag>
void run_dag(vsie_coupling_s* h, int op, int nrhs, const void* x, void* y, const void* u, void* z, cudaStream_t st,
             Dag&& dag) {
  ensure_streams(h);
  h->apply_calls += 1;
  if (h->timing == 2) {
    // timeline: the concurrent DAG launched eagerly, event pairs around every kernel
    cudaEvent_t o;
    VSIE_CHECK_CUDA(cudaEventCreate(&o));
    h->origins.push_back(o);
    VSIE_CHECK_CUDA(cudaEventRecord(o, st));
    h->trace_origin = o;
    Streams S = make_streams(h, st, true);
    const int64_t before = launch_counter();
    dag(S);
    h->apply_launches += launch_counter() - before;
    h->trace_call += 1;
    return;
  }
  auto capture = [&](const Streams& S, int64_t& launches) -> cudaGraph_t {
    const int64_t before = launch_counter();
    VSIE_CHECK_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t graph = nullptr;
    try {
      dag(S);
    } catch (...) {
      cudaStreamEndCapture(h->cap_stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    VSIE_CHECK_CUDA(cudaStreamEndCapture(h->cap_stream, &graph));
    launches = launch_counter() - before;
    return graph;
  };
  if (h->timing) {
    // per-kernel CUDA-event timing: the same DAG serialised on one stream, captured with
    // its event records into a one-shot graph so that host submission gaps do not enter
    // the per-kernel durations
    Streams S = make_streams(h, h->cap_stream, false);
    int64_t launches = 0;
    cudaGraph_t graph = capture(S, launches);
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    VSIE_CHECK_CUDA(e);
    e = cudaGraphLaunch(exec, st);
    cudaGraphExecDestroy(exec);
    VSIE_CHECK_CUDA(e);
    h->apply_launches += launches;
    return;
  }
  if (!graphs_enabled(h)) {
    Streams S = make_streams(h, st, true);
    const int64_t before = launch_counter();
    dag(S);
    h->apply_launches += launch_counter() - before;
    return;
  }
  GraphEntry* ge = nullptr;
  for (GraphEntry& g : h->graphs)
    if (g.op == op && g.nrhs == nrhs && g.x == x && g.y == y && g.u == u && g.z == z) ge = &g;
  if (!ge) {
    if (h->graphs.size() >= 16) {
      auto lru = std::min_element(h->graphs.begin(), h->graphs.end(),
                                  [](const GraphEntry& a, const GraphEntry& b) { return a.last_use < b.last_use; });
      cudaGraphExecDestroy(lru->exec);
      h->graphs.erase(lru);
    }
    GraphEntry g;
    g.op = op;
    g.nrhs = nrhs;
    g.x = x;
    g.y = y;
    g.u = u;
    g.z = z;
    Streams S = make_streams(h, h->cap_stream, true);
    cudaGraph_t graph = capture(S, g.launches);
    cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    VSIE_CHECK_CUDA(e);
    h->graphs.push_back(g);
    ge = &h->graphs.back();
  }
  ge->last_use = ++h->graph_clock;
  VSIE_CHECK_CUDA(cudaGraphLaunch(ge->exec, st));
  h->apply_launches += ge->launches;
}

// The GMRES pair with every contraction step as ONE launch over the three chi on a single
// stream (programmatic dependent launch between steps): G1^T, G2^T, G3^T (k_seg_gemv),
// G4 both ways (k_pair_g4), G3 (k_seg_gemv), G2, G1.  false if a step's shape is not
// supported by the batched kernels (the caller then runs the chain schedule).
bool pair_batched(vsie_coupling_s* h, const cplx* x, cplx* y, const cplx* u, cplx* z, bool cj, cudaStream_t st) {
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  int r1m = 1, r2m = 1, r3m = 1;
  for (int c = 0; c < 3; ++c) {
    r1m = std::max(r1m, h->ranks[c][0]);
    r2m = std::max(r2m, h->ranks[c][1]);
    r3m = std::max(r3m, h->ranks[c][2]);
  }
  if (r3m > pair_g4_max_rank() || h->shards.size() != 1 || h->comm) return false;
  Shard& s = h->shards[0];
  const int64_t n3l = s.n3loc();
  if (n3l == 0 || s.mloc() == 0) return false;
  for (int c = 0; c < 3; ++c)
    if (!seg_gemv_supported((int64_t)h->ranks[c][1] * n3l, h->ranks[c][2], s.g3b_ns)) return false;
  int w2_splits = 0;
  int64_t w2_stride = 0;
  const IoLayout L = voxel_layout(h);
  auto R = [&](int c, int j) { return (int64_t)h->ranks[c][j]; };
  cplx* part = h->partials.p;
  cplx* zws = h->zgemm_ws.p;
  const int64_t zcap = 3 * h->zgemm_ws_per_chi;
  {
    ReduceArgs r{};
    r.nbatch = 3;
    r.n1 = n1;
    r.ncol = (int64_t)n2 * n3l;
    r.cols_per_rhs = r.ncol;
    r.ld_rhs = L.ld;
    r.conj_u = cj;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      r.G1[c] = h->G1[c].p;
      r.u[c] = u + c * L.chi_stride;
      r.W1[c] = s.W1.p + c * r1m * n2 * n3l;
      r.r1[c] = (int)R(c, 0);
      bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l + (int64_t)n1 * n2 * n3l);
      fl += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l;
    }
    Scope sc(h, "adj_g1_reduce", bytes, fl, st);
    launch_reduce_g1(r, st);
  }
  {
    Zgemm zg{};
    zg.nbatch = 3;
    zg.ta = kT;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      zg.M[c] = R(c, 1); zg.N[c] = n3l; zg.K[c] = R(c, 0) * n2;
      zg.A[c] = h->G2[c].p; zg.lda[c] = R(c, 0) * n2;
      zg.B[c] = s.W1.p + c * r1m * n2 * n3l; zg.ldb[c] = R(c, 0) * n2;
      zg.C[c] = s.W2.p + c * r2m * n3l; zg.ldc[c] = R(c, 1);
      bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l + R(c, 0) * n2 * n3l);
      fl += 8 * R(c, 0) * n2 * R(c, 1) * n3l;
    }
    Scope sc(h, "adj_g2_zgemm", bytes, fl, st);
    if (w2_parts_on())
      w2_splits = launch_zgemm_dmma_parts(zg, zws, zcap, st, &w2_stride);
    else
      launch_zgemm_dmma(zg, zws, zcap, st);
  }
  SegGemv g{};
  g.nbatch = 3;
  g.nsb = s.g3b_ns;
  g.partials = part;
  g.rstride = r3m;
  int64_t b3 = 0;
  for (int c = 0; c < 3; ++c) {
    g.A[c] = s.G3b[c].p;
    g.x[c] = s.W2.p + c * r2m * n3l;
    g.xparts[c] = w2_splits;
    g.xpart[c] = zws + (int64_t)c * w2_splits * w2_stride;
    g.xpart_stride[c] = w2_stride;
    g.y[c] = s.z3.p + c * r3m;
    g.R[c] = R(c, 1) * n3l;
    g.C[c] = R(c, 2);
    b3 += 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]);
  }
  {
    Scope sc(h, "adj_g3_seg", b3, b3 / 2, st);
    VSIE_REQUIRE(launch_seg_gemv(g, true, st), VSIE_ERR_STATE, "pair_batched: G3 shape");
  }
  {
    PairG4 p{};
    p.nbatch = 3;
    p.C = s.mloc();
    p.x = x + s.cb;
    p.z = z + s.cb;
    p.conj_z = cj;
    p.partials = part;
    p.rstride = r3m;
    for (int c = 0; c < 3; ++c) {
      p.A[c] = s.G4[c].p;
      p.z3[c] = s.z3.p + c * r3m;
      p.y4[c] = s.y4.p + c * r3m;
      p.R[c] = R(c, 2);
    }
    Scope sc(h, "pair_g4_tma", 16 * (R(0, 2) + R(1, 2) + R(2, 2)) * (p.C + 2) + 16 * 2 * p.C,
             16 * (R(0, 2) + R(1, 2) + R(2, 2)) * p.C, st);
    VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), st), VSIE_ERR_STATE, "pair_batched: G4 shape");
  }
  for (int c = 0; c < 3; ++c) {
    g.x[c] = s.y4.p + c * r3m;
    g.y[c] = s.Y3.p + c * r2m * n3l;
    g.xparts[c] = 0;
  }
  {
    Scope sc(h, "fwd_g3_seg", b3, b3 / 2, st);
    VSIE_REQUIRE(launch_seg_gemv(g, false, st), VSIE_ERR_STATE, "pair_batched: G3 shape");
  }
  {
    Zgemm zg{};
    zg.nbatch = 3;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      zg.M[c] = R(c, 0) * n2; zg.N[c] = n3l; zg.K[c] = R(c, 1);
      zg.A[c] = h->G2[c].p; zg.lda[c] = R(c, 0) * n2;
      zg.B[c] = s.Y3.p + c * r2m * n3l; zg.ldb[c] = R(c, 1);
      zg.C[c] = s.Y2.p + c * r1m * n2 * n3l; zg.ldc[c] = R(c, 0) * n2;
      bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l + R(c, 0) * n2 * n3l);
      fl += 8 * R(c, 0) * n2 * R(c, 1) * n3l;
    }
    Scope sc(h, "fwd_g2_zgemm", bytes, fl, st);
    launch_zgemm_dmma(zg, zws, zcap, st);
  }
  {
    ExpandArgs e{};
    e.nbatch = 3;
    e.n1 = n1;
    e.ncol = (int64_t)n2 * n3l;
    e.cols_per_rhs = e.ncol;
    e.ld_rhs = L.ld;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      e.G1[c] = h->G1[c].p;
      e.Y2[c] = s.Y2.p + c * r1m * n2 * n3l;
      e.y[c] = y + c * L.chi_stride;
      e.r1[c] = (int)R(c, 0);
      bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l + (int64_t)n1 * n2 * n3l);
      fl += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l;
    }
    Scope sc(h, "fwd_g1_expand", bytes, fl, st);
    launch_expand_g1(e, st);
  }
  return true;
}

// the forward's G2 and G1 steps for the three chi as one batched launch each (Y3 formed)
// instead of per-chi chains; VSIE_FWD_TAIL_BATCHED=1
bool fwd_tail_batched_on() {
  static const int v = [] {
    const char* e = std::getenv("VSIE_FWD_TAIL_BATCHED");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

void fwd_tail_batched(vsie_coupling_s* h, const Ctx& X, Shard& s, cplx* y, cudaStream_t st) {
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  if (n3l == 0) return;
  {
    Zgemm zg{};
    zg.nbatch = 3;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      zg.M[c] = X.R(c, 0) * n2; zg.N[c] = n3l; zg.K[c] = X.R(c, 1);
      zg.A[c] = h->G2[c].p; zg.lda[c] = X.R(c, 0) * n2;
      zg.B[c] = s.Y3.p + c * X.r2m * n3l; zg.ldb[c] = X.R(c, 1);
      zg.C[c] = s.Y2.p + c * X.r1m * n2 * n3l; zg.ldc[c] = X.R(c, 0) * n2;
      bytes += 16 * (X.R(c, 0) * n2 * X.R(c, 1) + X.R(c, 1) * n3l + X.R(c, 0) * n2 * n3l);
      fl += 8 * X.R(c, 0) * n2 * X.R(c, 1) * n3l;
    }
    Scope sc(h, "fwd_g2_zgemm_b", bytes, fl, st);
    launch_zgemm_dmma(zg, h->zgemm_ws.p, 3 * h->zgemm_ws_per_chi, st);
  }
  {
    ExpandArgs e{};
    e.nbatch = 3;
    e.n1 = n1;
    e.ncol = (int64_t)n2 * n3l;
    e.cols_per_rhs = e.ncol;
    e.ld_rhs = X.L.ld;
    int64_t bytes = 0, fl = 0;
    for (int c = 0; c < 3; ++c) {
      e.G1[c] = h->G1[c].p;
      e.Y2[c] = s.Y2.p + c * X.r1m * n2 * n3l;
      e.y[c] = y + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
      e.r1[c] = (int)X.R(c, 0);
      bytes += 16 * ((int64_t)n1 * X.R(c, 0) + X.R(c, 0) * n2 * n3l + (int64_t)n1 * n2 * n3l);
      fl += 8 * (int64_t)n1 * X.R(c, 0) * n2 * n3l;
    }
    Scope sc(h, "fwd_g1_expand_b", bytes, fl, st);
    launch_expand_g1(e, st);
  }
}

// The coupling pair of one GMRES matvec of the hybrid system (Eq. 11 / 15: the body rows
// need Z_bc j_c, the conductor rows Z_bc^T j_b): y = Z x and z = Z^T u (Z^H u).  The
// transpose front (G1^T, G2^T, G3^T) runs first, so that both directions' G4 products
// share ONE stream of the largest core (k_gemv_nt); the forward finishes from y4.
void pair_dag(vsie_coupling_s* h, const cplx* x, cplx* y, const cplx* u, cplx* z, bool cj, const Streams& S) {
  Ctx X;
  X.h = h;
  X.k = 1;
  X.r1m = X.r2m = X.r3m = 1;
  for (int c = 0; c < 3; ++c) {
    X.r1m = std::max(X.r1m, h->ranks[c][0]);
    X.r2m = std::max(X.r2m, h->ranks[c][1]);
    X.r3m = std::max(X.r3m, h->ranks[c][2]);
  }
  X.r3stride = X.r3m;
  X.L = voxel_layout(h);
  const bool exchange = h->comm != nullptr || h->shards.size() > 1;
  const int64_t m = h->m, mp = ceil_div(m, h->world);
  if (pair_g4_mode() == 4 && pair_batched(h, x, y, u, z, cj, S.main)) return;
  if (pair_g4_mode() == 5 && !exchange && X.r3m <= pair_g4_max_rank()) {
    // overlap schedule: the forward's G4 pass (needs only x) streams while the transpose's
    // G1 / G2 steps compute in the chi chains; one pass over G3 serves both directions;
    // the transpose's G4 pass streams while the forward's G2 / G1 steps compute
    Shard& s = h->shards[0];
    const int64_t n3l = s.n3loc();
    bool ok = n3l > 0 && s.mloc() > 0;
    for (int c = 0; c < 3 && ok; ++c) ok = seg_gemv_supported(X.R(c, 1) * n3l, X.R(c, 2), s.g3b_ns);
    if (ok) {
      cplx* part2 = h->partials.p + 3 * h->partials_per_chi;   // not used by the chains
      fork(h, S);
      {
        PairG4 p{};
        p.nbatch = 3;
        p.C = s.mloc();
        p.x = x + s.cb;
        p.partials = part2;
        p.rstride = X.r3m;
        for (int c = 0; c < 3; ++c) {
          p.A[c] = s.G4[c].p;
          p.y4[c] = s.y4.p + c * X.r3stride;
          p.R[c] = X.R(c, 2);
        }
        Scope sc(h, "fwd_g4_tma", 16 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * (p.C + 1) + 16 * p.C,
                 8 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * p.C, S.main);
        VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), S.main), VSIE_ERR_STATE, "pair mode 5: G4 shape");
      }
      for (int c = 0; c < 3; ++c) {
        h->scope_chi = c;
        adj_front(X, s, c, u, cj, S.chi[c], nullptr, false, true);
      }
      h->scope_chi = -1;
      join(h, S);
      {
        SegGemv g{};
        g.nbatch = 3;
        g.nsb = s.g3b_ns;
        g.partials = part2;
        g.rstride = X.r3m;
        int64_t bytes = 0;
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G3b[c].p;
          g.x[c] = s.y4.p + c * X.r3stride;
          g.y[c] = s.Y3.p + c * X.r2m * n3l;
          g.xt[c] = s.W2.p + c * X.r2m * n3l;
          g.yt[c] = s.z3.p + c * X.r3stride;
          g.xparts[c] = 0;
          g.R[c] = X.R(c, 1) * n3l;
          g.C[c] = X.R(c, 2);
          bytes += 16 * (g.R[c] * g.C[c] + 2 * (g.R[c] + g.C[c]));
        }
        Scope sc(h, "g3_seg_both", bytes, bytes, S.main);
        VSIE_REQUIRE(launch_seg_gemv_mode(g, 3, S.main), VSIE_ERR_STATE, "pair mode 5: G3 shape");
      }
      fork(h, S);
      {
        PairG4 p{};
        p.nbatch = 3;
        p.C = s.mloc();
        p.z = z + s.cb;
        p.conj_z = cj;
        p.partials = part2;
        p.rstride = X.r3m;
        for (int c = 0; c < 3; ++c) {
          p.A[c] = s.G4[c].p;
          p.z3[c] = s.z3.p + c * X.r3stride;
          p.R[c] = X.R(c, 2);
        }
        Scope sc(h, "adj_g4_tma", 16 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * (p.C + 1) + 16 * p.C,
                 8 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * p.C, S.main);
        VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), S.main), VSIE_ERR_STATE, "pair mode 5: G4 shape");
      }
      for (int c = 0; c < 3; ++c) {
        h->scope_chi = c;
        fwd_rest(X, s, c, y, S.chi[c], nullptr, false);
      }
      h->scope_chi = -1;
      join(h, S);
      return;
    }
  }
  if (pair_g4_mode() == 3 && !exchange) {
    // both directions as six independent chains (transpose chains on S.chi, forward chains
    // on S.chi2, separate workspaces): G4 is read twice but no chain waits for another
    Ctx XA = X;
    XA.ws = 3;
    Shard& s = h->shards[0];
    fork(h, S, true);
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      adj_front(XA, s, c, u, cj, S.chi[c]);
      adj_g4(XA, s, c, S.chi[c]);
      fwd_g4(X, s, c, x, S.chi2[c]);
      fwd_rest(X, s, c, y, S.chi2[c]);
    }
    h->scope_chi = -1;
    join(h, S, true);
    adj_sum_chi(X, s, z + s.cb, m, cj, S.main);
    return;
  }
  // mode 2: the G3 and G4 steps as batched TMA-streamed launches on the main stream
  // (both directions), the G1 / G2 steps as per-chi chains around them
  bool seg = pair_g4_mode() == 2 && seg_g3_on();
  for (Shard& s : h->shards)
    for (int c = 0; c < 3 && seg; ++c)
      seg = seg_gemv_supported(X.R(c, 1) * s.n3loc(), X.R(c, 2), s.g3b_ns) && s.n3loc() > 0;
  // transpose front entirely in the chi chains (G1^T, G2^T and a small-ring G3^T pass per
  // chi), VSIE_ADJ_CHAIN_SEG=1
  const bool adj_chain = seg && adj_chain_seg_on() && !exchange && g2t_on() && !reduce_tma_on() &&
                         !adj_fused_on();
  if (adj_chain) {
    Shard& s = h->shards[0];
    const int64_t n3l = s.n3loc();
    fork(h, S);
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      adj_front(X, s, c, u, cj, S.chi[c], nullptr, false, true, false);   // G1^T only
      launch_g2t_shard(h, X, s, S.chi[c], c);
      SegGemv g{};
      g.nbatch = 1;
      g.nsb = s.g3b_ns;
      g.partials = X.partials(c);   // per chain: the chains run concurrently
      g.rstride = X.r3m;
      g.A[0] = s.G3b[c].p;
      g.x[0] = s.W2.p + c * X.r2m * n3l;
      g.xparts[0] = 0;
      g.y[0] = s.z3.p + c * X.r3stride;
      g.R[0] = X.R(c, 1) * n3l;
      g.C[0] = X.R(c, 2);
      const int64_t bytes = 16 * (g.R[0] * g.C[0] + g.R[0] + g.C[0]);
      Scope sc(h, "adj_g3_seg_chi", bytes, bytes / 2, S.chi[c]);
      VSIE_REQUIRE(launch_seg_gemv_mode(g, 2, S.chi[c], true), VSIE_ERR_STATE, "pair: G3 shape");
    }
    h->scope_chi = -1;
    join(h, S);
    fork(h, S);
  } else {
    // the fused G1^T + G2^T kernel (one launch over the three chi) replaces the chains
    const bool fused_front = seg && adj_fused_on() && adj_front_supported(h->grid.n[0], X.r1m);
    if (fused_front) {
      const int n2 = h->grid.n[1];
      for (Shard& s : h->shards) {
        const int64_t n3l = s.n3loc();
        AdjFrontArgs f{};
        f.nbatch = 3;
        f.n1 = h->grid.n[0];
        f.n2 = n2;
        f.n3l = (int)n3l;
        f.conj_u = cj;
        f.w2p_stride = (int64_t)X.r2m * n3l;
        int64_t bytes = 0, fl = 0;
        for (int c = 0; c < 3; ++c) {
          f.G1[c] = h->G1[c].p;
          f.G2[c] = h->G2[c].p;
          f.u[c] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
          f.W2p[c] = s.W2p.p + c * (int64_t)((n2 + 7) / 8) * X.r2m * n3l;
          f.W2[c] = s.W2.p + c * X.r2m * n3l;
          f.r1[c] = (int)X.R(c, 0);
          f.r2[c] = (int)X.R(c, 1);
          h->w2_parts[c] = 0;
          bytes += 16 * ((int64_t)f.n1 * X.R(c, 0) + X.R(c, 0) * n2 * X.R(c, 1) + (int64_t)f.n1 * n2 * n3l +
                         X.R(c, 1) * n3l);
          fl += 8 * ((int64_t)f.n1 * X.R(c, 0) * n2 * n3l + X.R(c, 0) * n2 * X.R(c, 1) * n3l);
        }
        Scope sc(h, "adj_g12_fused", bytes, fl, S.main);
        launch_adj_front(f, S.main);
      }
    } else {
      // W1 = G1^T u for the three chi as one TMA-streamed launch when supported, then the
      // G2^T steps as per-chi chains
      bool g1_done = false;
      if (seg && reduce_tma_on() && reduce_tma_fits(h->grid.n[0], X.r1m)) {
        g1_done = true;
        for (Shard& s : h->shards) {
          const int64_t n3l = s.n3loc();
          ReduceArgs r{};
          r.nbatch = 3;
          r.n1 = h->grid.n[0];
          r.ncol = (int64_t)h->grid.n[1] * n3l;
          r.cols_per_rhs = r.ncol;
          r.ld_rhs = X.L.ld;
          r.conj_u = cj;
          int64_t bytes = 0, fl = 0;
          for (int c = 0; c < 3; ++c) {
            r.G1[c] = h->G1[c].p;
            r.u[c] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
            r.W1[c] = s.W1.p + c * X.r1m * h->grid.n[1] * n3l;
            r.r1[c] = (int)X.R(c, 0);
            bytes += 16 * ((int64_t)r.n1 * X.R(c, 0) + X.R(c, 0) * r.ncol + (int64_t)r.n1 * r.ncol);
            fl += 8 * (int64_t)r.n1 * X.R(c, 0) * r.ncol;
          }
          Scope sc(h, "adj_g1_reduce_tma", bytes, fl, S.main);
          g1_done = g1_done && n3l > 0 && launch_reduce_g1_tma(r, S.main);
        }
        VSIE_REQUIRE(g1_done || h->shards.size() == 1, VSIE_ERR_STATE, "reduce_tma on a partial shard set");
      }
      const bool g2b = seg && g2t_on() && X.k == 1;
      const bool g2chain = g2b && !g1_done && g2t_chain_on();
      if (!(g1_done && g2b)) {
        fork(h, S);
        for (int c = 0; c < 3; ++c) {
          h->scope_chi = c;
          for (Shard& s : h->shards) {
            adj_front(X, s, c, u, cj, S.chi[c], nullptr, !seg, !g1_done, !g2b);
            if (g2chain) launch_g2t_shard(h, X, s, S.chi[c], c);   // this chi's G2^T in its chain
          }
        }
        h->scope_chi = -1;
        if (g2b) join(h, S);
      }
      if (g2b && !g2chain) {
        for (Shard& s : h->shards) launch_g2t_shard(h, X, s, S.main);
      }
    }
    if (seg) {
      if (!fused_front && !(seg && g2t_on())) join(h, S);
      for (Shard& s : h->shards) {
        const int64_t n3l = s.n3loc();
        SegGemv g{};
        g.nbatch = 3;
        g.nsb = s.g3b_ns;
        g.partials = X.partials(0);
        g.rstride = X.r3m;
        int64_t bytes = 0;
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G3b[c].p;
          g.x[c] = s.W2.p + c * X.r2m * n3l;
          g.xparts[c] = h->shards.size() == 1 ? h->w2_parts[c] : 0;
          g.xpart[c] = X.zws(c);
          g.xpart_stride[c] = h->w2_part_stride[c];
          g.y[c] = s.z3.p + c * X.r3stride;
          g.R[c] = X.R(c, 1) * n3l;
          g.C[c] = X.R(c, 2);
          bytes += 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]);
        }
        bool ok;
        {
          Scope sc(h, "adj_g3_seg", bytes, bytes / 2, S.main);
          ok = n3l > 0 && launch_seg_gemv(g, true, S.main);
        }
        if (!ok) {
          // unsupported shape: the per-chi column GEMVs
          for (int c = 0; c < 3; ++c) {
            cplx* z3 = s.z3.p + c * X.r3stride;
            if (n3l == 0) {
              VSIE_CHECK_CUDA(cudaMemsetAsync(z3, 0, X.r3stride * sizeof(cplx), S.main));
              continue;
            }
            GemvT t{};
            t.nbatch = 1;
            t.A[0] = s.G3[c].p;
            t.x[0] = g.x[c];
            t.y[0] = z3;
            t.R[0] = g.R[c];
            t.C[0] = g.C[c];
            Scope sc(h, "adj_g3_gemv", 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]), 8 * g.R[c] * g.C[c], S.main);
            launch_gemv_t(t, X.partials(c), h->partials_per_chi, kMaxSplits, S.main);
          }
        }
      }
      if (exchange) combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
      fork(h, S);
    } else if (exchange) {
      join(h, S);
      combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
      fork(h, S);
    }
  }
  if (pair_g4_mode() == 2 && seg && g4_chain_on() && !exchange && X.r3m <= pair_g4_max_rank()) {
    // per chi in its chain: the G4 pass (both products, small ring), the G3 pass, G2 and G1
    // -- chi c's G2 / G1 kernels run beside chi c + 1's G4 / G3 streams; Eq. 18 sum at the end
    Shard& s = h->shards[0];
    const int64_t n3l = s.n3loc(), ldz = s.zpart.n / 3;
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      PairG4 p{};
      p.nbatch = 1;
      p.C = s.mloc();
      p.x = x + s.cb;
      p.z = s.zpart.p + c * ldz;
      p.partials = X.partials(c);
      p.rstride = X.r3m;
      p.small_ring = true;
      p.A[0] = s.G4[c].p;
      p.z3[0] = s.z3.p + c * X.r3stride;
      p.y4[0] = s.y4.p + c * X.r3stride;
      p.R[0] = X.R(c, 2);
      {
        Scope sc(h, "pair_g4_chi", 16 * X.R(c, 2) * (p.C + 2) + 16 * 2 * p.C, 16 * X.R(c, 2) * p.C, S.chi[c]);
        VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), S.chi[c]), VSIE_ERR_STATE, "pair: G4 shape");
      }
      SegGemv g{};
      g.nbatch = 1;
      g.nsb = s.g3b_ns;
      g.A[0] = s.G3b[c].p;
      g.x[0] = s.y4.p + c * X.r3stride;
      g.y[0] = s.Y3.p + c * X.r2m * n3l;
      g.R[0] = X.R(c, 1) * n3l;
      g.C[0] = X.R(c, 2);
      {
        const int64_t bytes = 16 * (g.R[0] * g.C[0] + g.R[0] + g.C[0]);
        Scope sc(h, "fwd_g3_seg_chi", bytes, bytes / 2, S.chi[c]);
        VSIE_REQUIRE(launch_seg_gemv_mode(g, 1, S.chi[c], true), VSIE_ERR_STATE, "pair: G3 shape");
      }
      fwd_rest(X, s, c, y, S.chi[c], nullptr, false);
    }
    h->scope_chi = -1;
    join(h, S);
    adj_sum_chi(X, s, z + s.cb, m, cj, S.main);
    return;
  }
  bool z_done = false;
  if (pair_g4_mode() == 2) {
    // one TMA-streamed pass over the three G4 cores: y4 (all chi) and z = sum_chi G4^T z3
    join(h, S);
    bool ok = true;
    for (Shard& s : h->shards) {
      PairG4 g{};
      g.nbatch = 3;
      g.C = s.mloc();
      g.x = x + s.cb;
      g.z = h->comm ? h->gather_buf.p + (int64_t)h->world * mp : z + s.cb;
      g.conj_z = cj;
      g.partials = X.partials(0);
      g.rstride = X.r3m;
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G4[c].p;
        g.z3[c] = s.z3.p + c * X.r3stride;
        g.y4[c] = s.y4.p + c * X.r3stride;
        g.R[c] = X.R(c, 2);
      }
      if (g.C == 0) {
        VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p, 0, 3 * X.r3stride * sizeof(cplx), S.main));
        continue;
      }
      Scope sc(h, "pair_g4_tma", 16 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * (g.C + 2) + 16 * 2 * g.C,
               16 * (X.R(0, 2) + X.R(1, 2) + X.R(2, 2)) * g.C, S.main);
      ok = ok && launch_pair_g4(g, sm_count_dev(), S.main);
    }
    VSIE_REQUIRE(ok || h->shards.size() == 1, VSIE_ERR_STATE, "pair_g4 unsupported on a multi-shard handle");
    z_done = ok;
    if (z_done && exchange) combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
    if (z_done && seg && !(fwd_chain_seg_on(h) && !fwd_tail_batched_on() && !g2n_on())) {
      for (Shard& s : h->shards) {
        const int64_t n3l = s.n3loc();
        if (n3l == 0) continue;
        SegGemv g{};
        g.nbatch = 3;
        g.nsb = s.g3b_ns;
        int64_t bytes = 0;
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G3b[c].p;
          g.x[c] = s.y4.p + c * X.r3stride;
          g.y[c] = s.Y3.p + c * X.r2m * n3l;
          g.R[c] = X.R(c, 1) * n3l;
          g.C[c] = X.R(c, 2);
          bytes += 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]);
        }
        bool ok3;
        {
          Scope sc(h, "fwd_g3_seg", bytes, bytes / 2, S.main);
          ok3 = launch_seg_gemv(g, false, S.main);
        }
        if (!ok3) {
          for (int c = 0; c < 3; ++c) {
            GemvN t{};
            t.nbatch = 1;
            t.A[0] = s.G3[c].p;
            t.x[0] = g.x[c];
            t.y[0] = g.y[c];
            t.R[0] = g.R[c];
            t.C[0] = g.C[c];
            Scope sc(h, "fwd_g3_gemv", 16 * (g.R[c] * g.C[c] + g.R[c] + g.C[c]), 8 * g.R[c] * g.C[c], S.main);
            launch_gemv_n(t, X.partials(c), h->partials_per_chi, kMaxSplits, S.main);
          }
        }
      }
    }
    fork(h, S);
  }
  if (!z_done) {
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) {
      const int64_t ml = s.mloc();
      const int64_t ldz = s.zpart.n / 3;   // nrhs_max columns per chi block; single RHS here
      if (ml == 0) {
        VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p + c * X.r3stride, 0, X.r3stride * sizeof(cplx), S.chi[c]));
        continue;
      }
      const int64_t r3 = X.R(c, 2);
      GemvNT g{};
      g.nbatch = 1;
      g.A[0] = s.G4[c].p;
      g.x[0] = x + s.cb;
      g.z3[0] = s.z3.p + c * X.r3stride;
      g.z[0] = s.zpart.p + c * ldz;
      g.y4[0] = s.y4.p + c * X.r3stride;
      g.R[0] = r3;
      g.C[0] = ml;
      bool fused;
      {
        Scope sc(h, "pair_g4_nt", 16 * (r3 * ml + 2 * ml + 2 * r3), 16 * r3 * ml, S.chi[c]);
        fused = launch_gemv_nt(g, X.partials(c), h->partials_per_chi, S.chi[c]);
      }
      if (!fused) {   // r3 > 320: the two G4 products as separate passes
        fwd_g4(X, s, c, x, S.chi[c]);
        adj_g4(X, s, c, S.chi[c]);
      }
    }
  }
  if (exchange) {
    join(h, S);
    combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
    fork(h, S);
  }
  }   // !z_done
  if (z_done && seg && fwd_tail_batched_on()) {
    for (Shard& s : h->shards) fwd_tail_batched(h, X, s, y, S.main);
  } else if (z_done && seg && g2n_on()) {
    // Y2 = G2 Y3 for the three chi in one launch (k_g2n), then the G1 expansions per chi
    join(h, S);
    for (Shard& s : h->shards) launch_g2n_shard(h, X, s, S.main);
    fork(h, S);
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) fwd_expand(X, s, c, y, S.chi[c]);
    }
  } else {
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) {
        if (z_done && seg && fwd_chain_seg_on(h) && !fwd_tail_batched_on() && !g2n_on()) {
          // this chi's G3 pass in its chain (small ring: the chain's G2 / G1 kernels of the
          // previous chi fit beside it on the SMs)
          const int64_t n3l = s.n3loc();
          if (n3l == 0) continue;
          SegGemv g{};
          g.nbatch = 1;
          g.nsb = s.g3b_ns;
          g.A[0] = s.G3b[c].p;
          g.x[0] = s.y4.p + c * X.r3stride;
          g.y[0] = s.Y3.p + c * X.r2m * n3l;
          g.R[0] = X.R(c, 1) * n3l;
          g.C[0] = X.R(c, 2);
          const int64_t bytes = 16 * (g.R[0] * g.C[0] + g.R[0] + g.C[0]);
          {
            Scope sc(h, "fwd_g3_seg_chi", bytes, bytes / 2, S.chi[c]);
            VSIE_REQUIRE(launch_seg_gemv_mode(g, 1, S.chi[c], true), VSIE_ERR_STATE, "pair: G3 shape");
          }
        }
        fwd_rest(X, s, c, y, S.chi[c], nullptr, !(z_done && seg));
      }
    }
  }
  h->scope_chi = -1;
  join(h, S);
  for (Shard& s : h->shards) {
    if (z_done) break;
    if (h->comm)
      adj_sum_chi(X, s, h->gather_buf.p + (int64_t)h->world * mp, mp, cj, S.main);
    else
      adj_sum_chi(X, s, z + s.cb, m, cj, S.main);
  }
  if (h->comm) {
    Scope sc(h, "nccl_allgather", 0, 0, S.main);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) VSIE_CHECK_CUDA(cudaMemsetAsync(seg + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), S.main));
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p), 2 * (size_t)mp,
                       S.main);
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(z + cb, m, h->gather_buf.p + (int64_t)p * mp, mp, ce - cb, 1, S.main);
    }
  }
}

}  // namespace

void apply(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st) {
  VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "bad op");
  VSIE_REQUIRE(nrhs >= 1 && nrhs <= h->nrhs_max, VSIE_ERR_ARG, "nrhs out of range");
  VSIE_REQUIRE(x != nullptr && y != nullptr, VSIE_ERR_ARG, "x / y is NULL");
  run_dag(h, op, nrhs, x, y, nullptr, nullptr, st, [&](const Streams& S) { apply_dag(h, x, y, op, nrhs, S); });
}

void apply_pair(vsie_coupling_s* h, const cplx* x, cplx* y, const cplx* u, cplx* z, int adj_op, cudaStream_t st) {
  VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
  VSIE_REQUIRE(adj_op == VSIE_OP_T || adj_op == VSIE_OP_C, VSIE_ERR_ARG, "adj_op must be OP_T or OP_C");
  VSIE_REQUIRE(x && y && u && z, VSIE_ERR_ARG, "x / y / u / z is NULL");
  if (h->apply_mode != 0) {   // the fused pair is built on the chain schedule
    apply(h, x, y, VSIE_OP_N, 1, st);
    apply(h, u, z, adj_op, 1, st);
    return;
  }
  run_dag(h, 100 + adj_op, 1, x, y, u, z, st,
          [&](const Streams& S) { pair_dag(h, x, y, u, z, adj_op == VSIE_OP_C, S); });
}

}  // namespace vsie
