// The TT apply of Z_bc: forward y = Z x (Eq. 17) and plain /
// conjugate transpose z = Z^T u, Z^H u (Eqs. 18-19), and the GMRES coupling pair
// (both in one call), orchestrated over the kernels of pairg4.cu / segemv.cu / g2t.cu /
// ttapply.cu / linalg.cu.
//
// Each chi component is an independent TT.  The streaming steps on the two large
// cores (G4: r3 x m, G3: (r2 n3) x r3) run as ONE TMA-streamed launch over the three chi
// (k_pair_g4, k_seg_gemv: every CTA owns the same column / row range of every chi, the
// Eq. 18 sum over chi is formed inside the G4 pass); the compute-bound G1 / G2 steps run as
// three concurrent per-chi chains around them.  The whole fork/join DAG is captured once per
// (op, pointers) as a CUDA graph and replayed on the caller's stream; kernels are launched
// with programmatic dependent launch.  With the slab partition (SURVEY §8e design iii) the
// DAG joins around the cross-rank combines of y4 / z3 and the allgather of z.
//
// The GMRES pair (Eq. 11 / 15 rows: Z_bc j_c and Z_bc^T j_b in one matvec) has two
// schedules; the one that moves fewer bytes is chosen from the ranks:
//   G4-shared: transpose front (G1^T, G2^T, G3^T) first, then ONE pass over G4 for both
//              y4 = G4 x and z = sum_chi G4^T z3, then the forward's G3 / G2 / G1 steps:
//              G4 read once, G3 twice (cfgs 2 / 4: |G4| > |G3|);
//   G3-shared: forward G4 pass beside the transpose's G1^T chains, ONE pass over G3 for both
//              Y3 = G3 y4 and z3 = G3^T W2, then the transpose's G4 pass beside the
//              forward's G2 / G1 chains: G3 read once, G4 twice (cfgs 3 / 5: |G3| > |G4|).
// A GMRES step cannot read both once: the forward's G3 product needs the whole G4 pass and
// the transpose's G4 product needs the whole G3 pass.
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
  bool exchange() const { return h->comm != nullptr || h->shards.size() > 1; }
};

Ctx make_ctx(vsie_coupling_s* h, int nrhs) {
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
  return X;
}

constexpr int kMaxSplits = 256;

// ------------------------------------------------------------------ per-chi chain steps
// (block RHS, and the single-RHS fallback when a TMA pass does not support the shape)

// y4 = G4[:, owned] x[owned], partial per shard
void fwd_g4(const Ctx& X, Shard& s, int c, const cplx* x, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  cplx* y4 = s.y4.p + c * X.r3stride;
  if (s.mloc() == 0) {
    VSIE_CHECK_CUDA(cudaMemsetAsync(y4, 0, X.r3stride * sizeof(cplx), st));
    return;
  }
  const int64_t r3 = X.R(c, 2), ml = s.mloc();
  if (k == 1) {
    GemvN g{};
    g.nbatch = 1;
    g.A[0] = s.G4[c].p;
    g.x[0] = x + s.cb;
    g.y[0] = y4;
    g.R[0] = r3;
    g.C[0] = ml;
    Scope sc(h, "fwd_g4_gemv", 16 * (r3 * ml + ml + r3), 8 * r3 * ml, st);
    launch_gemv_n(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
    return;
  }
  Zgemm z{};
  z.M[0] = r3; z.N[0] = k; z.K[0] = ml;
  z.A[0] = s.G4[c].p; z.lda[0] = r3;
  z.B[0] = x + s.cb; z.ldb[0] = h->m;
  z.C[0] = y4; z.ldc[0] = r3;
  Scope sc(h, "fwd_g4_zgemm", 16 * (r3 * ml + (ml + r3) * k), 8 * r3 * ml * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
}

// Y3 = G3 y4 on the owned planes
void fwd_g3(const Ctx& X, Shard& s, int c, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int64_t n3l = s.n3loc(), r2 = X.R(c, 1), r3 = X.R(c, 2);
  cplx* y4 = s.y4.p + c * X.r3stride;
  cplx* Y3 = s.Y3.p + c * X.r2m * n3l * k;
  if (k == 1) {
    GemvN g{};
    g.nbatch = 1;
    g.A[0] = s.G3[c].p;
    g.x[0] = y4;
    g.y[0] = Y3;
    g.R[0] = r2 * n3l;
    g.C[0] = r3;
    Scope sc(h, "fwd_g3_gemv", 16 * (r2 * n3l * r3 + r2 * n3l + r3), 8 * r2 * n3l * r3, st);
    launch_gemv_n(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
    return;
  }
  Zgemm z{};
  z.M[0] = r2 * n3l; z.N[0] = k; z.K[0] = r3;
  z.A[0] = s.G3[c].p; z.lda[0] = r2 * n3l;
  z.B[0] = y4; z.ldb[0] = r3;
  z.C[0] = Y3; z.ldc[0] = r2 * n3l;
  Scope sc(h, "fwd_g3_zgemm", 16 * (r2 * n3l * r3 + (r2 * n3l + r3) * k), 8 * r2 * n3l * r3 * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
}

// Y2 = G2 Y3 of one chi
void fwd_g2(const Ctx& X, Shard& s, int c, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc(), r1 = X.R(c, 0), r2 = X.R(c, 1);
  Zgemm z{};
  z.M[0] = r1 * n2; z.N[0] = n3l * k; z.K[0] = r2;
  z.A[0] = h->G2[c].p; z.lda[0] = r1 * n2;
  z.B[0] = s.Y3.p + c * X.r2m * n3l * k; z.ldb[0] = r2;
  z.C[0] = s.Y2.p + c * X.r1m * n2 * n3l * k; z.ldc[0] = r1 * n2;
  Scope sc(h, "fwd_g2_zgemm", 16 * (r1 * n2 * r2 + r2 * n3l * k + r1 * n2 * n3l * k), 8 * r1 * n2 * r2 * n3l * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
}

// y = G1 Y2 of the chi [c0, c0 + nb) in one launch
void fwd_g1(const Ctx& X, Shard& s, int c0, int nb, cplx* y, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  ExpandArgs e{};
  e.nbatch = nb;
  e.n1 = n1;
  e.ncol = (int64_t)n2 * n3l * k;
  e.cols_per_rhs = (int64_t)n2 * n3l;
  e.ld_rhs = X.L.ld;
  int64_t r1s = 0;
  for (int i = 0; i < nb; ++i) {
    const int c = c0 + i;
    e.G1[i] = h->G1[c].p;
    e.Y2[i] = s.Y2.p + c * X.r1m * n2 * n3l * k;
    e.y[i] = y + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    e.r1[i] = (int)X.R(c, 0);
    r1s += X.R(c, 0);
  }
  Scope sc(h, "fwd_g1_expand", 16 * ((int64_t)n1 * r1s + r1s * n2 * n3l * k + (int64_t)nb * n1 * n2 * n3l * k),
           8 * (int64_t)n1 * r1s * n2 * n3l * k, st);
  launch_expand_g1(e, st);
}

// the forward's compute-bound tail of one chi: Y2 = G2 Y3, y = G1 Y2
void fwd_tail(const Ctx& X, Shard& s, int c, cplx* y, cudaStream_t st) {
  fwd_g2(X, s, c, st);
  fwd_g1(X, s, c, 1, y, st);
}

// W1 = G1^T u, conj(u) for op C
void adj_g1(const Ctx& X, Shard& s, int c, const cplx* u, bool cj, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc(), r1 = X.R(c, 0);
  ReduceArgs r{};
  r.nbatch = 1;
  r.n1 = n1;
  r.ncol = (int64_t)n2 * n3l * k;
  r.cols_per_rhs = (int64_t)n2 * n3l;
  r.ld_rhs = X.L.ld;
  r.conj_u = cj;
  r.G1[0] = h->G1[c].p;
  r.u[0] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
  r.W1[0] = s.W1.p + c * X.r1m * n2 * n3l * k;
  r.r1[0] = (int)r1;
  Scope sc(h, "adj_g1_reduce", 16 * ((int64_t)n1 * r1 + r1 * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k),
           8 * (int64_t)n1 * r1 * n2 * n3l * k, st);
  launch_reduce_g1(r, st);
}

// W1 = G1^T u for the three chi of one shard in one launch (single RHS)
void adj_g1_batched(const Ctx& X, Shard& s, const cplx* u, bool cj, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
  ReduceArgs r{};
  r.nbatch = 3;
  r.n1 = n1;
  r.ncol = (int64_t)n2 * n3l;
  r.cols_per_rhs = r.ncol;
  r.ld_rhs = X.L.ld;
  r.conj_u = cj;
  int64_t r1s = 0;
  for (int c = 0; c < 3; ++c) {
    r.G1[c] = h->G1[c].p;
    r.u[c] = u + c * X.L.chi_stride + shard_voxel_offset(h, s, X.L);
    r.W1[c] = s.W1.p + c * X.r1m * n2 * n3l;
    r.r1[c] = (int)X.R(c, 0);
    r1s += X.R(c, 0);
  }
  Scope sc(h, "adj_g1_reduce", 16 * ((int64_t)n1 * r1s + r1s * n2 * n3l + 3LL * n1 * n2 * n3l),
           8 * (int64_t)n1 * r1s * n2 * n3l, st);
  launch_reduce_g1(r, st, true);
}

// W2 = G2^T W1 of one chi as a split-K ZGEMM (block RHS)
void adj_g2(const Ctx& X, Shard& s, int c, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc(), r1 = X.R(c, 0), r2 = X.R(c, 1);
  Zgemm z{};
  z.ta = kT;
  z.M[0] = r2; z.N[0] = n3l * k; z.K[0] = r1 * n2;
  z.A[0] = h->G2[c].p; z.lda[0] = r1 * n2;
  z.B[0] = s.W1.p + c * X.r1m * n2 * n3l * k; z.ldb[0] = r1 * n2;
  z.C[0] = s.W2.p + c * X.r2m * n3l * k; z.ldc[0] = r2;
  Scope sc(h, "adj_g2_zgemm", 16 * (r1 * n2 * r2 + r2 * n3l * k + r1 * n2 * n3l * k), 8 * r1 * n2 * r2 * n3l * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
}

// z3 = G3^T W2, partial per shard
void adj_g3(const Ctx& X, Shard& s, int c, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  const int k = X.k;
  const int64_t n3l = s.n3loc(), r2 = X.R(c, 1), r3 = X.R(c, 2);
  cplx* W2 = s.W2.p + c * X.r2m * n3l * k;
  cplx* z3 = s.z3.p + c * X.r3stride;
  if (k == 1) {
    GemvT g{};
    g.nbatch = 1;
    g.A[0] = s.G3[c].p;
    g.x[0] = W2;
    g.y[0] = z3;
    g.R[0] = r2 * n3l;
    g.C[0] = r3;
    Scope sc(h, "adj_g3_gemv", 16 * (r2 * n3l * r3 + r2 * n3l + r3), 8 * r2 * n3l * r3, st);
    launch_gemv_t(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
    return;
  }
  Zgemm z{};
  z.ta = kT;
  z.M[0] = r3; z.N[0] = k; z.K[0] = r2 * n3l;
  z.A[0] = s.G3[c].p; z.lda[0] = r2 * n3l;
  z.B[0] = W2; z.ldb[0] = r2 * n3l;
  z.C[0] = z3; z.ldc[0] = r3;
  Scope sc(h, "adj_g3_zgemm", 16 * (r2 * n3l * r3 + (r2 * n3l + r3) * k), 8 * r2 * n3l * r3 * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
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
    Scope sc(h, "adj_g4_gemv", 16 * (r3 * ml + r3 + ml), 8 * r3 * ml, st);
    launch_gemv_t(g, X.partials(c), h->partials_per_chi, kMaxSplits, st);
    return;
  }
  Zgemm z{};
  z.ta = kT;
  z.M[0] = ml; z.N[0] = k; z.K[0] = r3;
  z.A[0] = s.G4[c].p; z.lda[0] = r3;
  z.B[0] = z3; z.ldb[0] = r3;
  z.C[0] = zp; z.ldc[0] = ldz;
  Scope sc(h, "adj_g4_zgemm", 16 * (r3 * ml + (r3 + ml) * k), 8 * r3 * ml * k, st);
  launch_zgemm_dmma(z, X.zws(c), h->zgemm_ws_per_chi, st);
}

// Eq. 18: z[owned] = sum_chi z_chi (fixed order), conj for op C
void adj_sum_chi(const Ctx& X, Shard& s, cplx* zout, int64_t ldz_out, bool cj, cudaStream_t st) {
  const int64_t ml = s.mloc();
  if (ml == 0) return;
  const int64_t ldz = s.zpart.n / (3 * X.k);
  Scope sc(X.h, "adj_sum_chi", 16 * 4 * ml * X.k, 0, st);
  launch_sum3(s.zpart.p, ldz * X.k, ldz, ml, X.k, zout, ldz_out, cj, st);
}

// ------------------------------------------------------------------ cross-rank combine
// sum the per-shard partial vectors (3 r3max nrhs) across ranks / loopback shards
void combine_r3(vsie_coupling_s* h, DevBuf<cplx> Shard::*buf, int64_t n, cudaStream_t st) {
  if (h->comm) {
    Scope sc(h, "comm_allreduce", 0, 0, st);
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

// where a shard writes its owned columns of z: the caller's z (one process) or the local
// segment of the allgather staging buffer ([mp x k], ld mp; multi-process)
int64_t seg_len(vsie_coupling_s* h) { return ceil_div(h->m, h->world); }
cplx* z_dest(vsie_coupling_s* h, const Shard& s, cplx* z, int k) {
  return h->comm ? h->gather_buf.p + (int64_t)h->world * seg_len(h) * k : z + s.cb;
}
int64_t z_ld(vsie_coupling_s* h) { return h->comm ? seg_len(h) : h->m; }

// multi-process: allgather of the column segments -> z replicated on every rank
void gather_z(vsie_coupling_s* h, cplx* z, int k, cudaStream_t st) {
  if (!h->comm) return;
  const int64_t m = h->m, mp = seg_len(h);
  cplx* seg = h->gather_buf.p + (int64_t)h->world * mp * k;
  const Shard& s = h->shards[0];
  Scope sc(h, "comm_allgather", 0, 0, st);
  for (int j = 0; j < k && s.mloc() < mp; ++j)
    VSIE_CHECK_CUDA(cudaMemsetAsync(seg + mp * j + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), st));
  h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p),
                     2 * (size_t)mp * k, st);
  for (int p = 0; p < h->world; ++p) {
    const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
    copy2d(z + cb, m, h->gather_buf.p + (int64_t)p * mp * k, mp, ce - cb, k, st);
  }
}

// ------------------------------------------------------------------ streams: fork / join
void ensure_streams(vsie_coupling_s* h) {
  if (h->chi_stream[0]) return;
  // chain chi gets stream priority rank chi (0 highest): the block scheduler then runs
  // chain 0 at full width and lets chains 1, 2 fill its ramp / tail / dependency bubbles
  int least = 0, greatest = 0;
  VSIE_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  for (int c = 0; c < 3; ++c) {
    const int prio = std::min(least, greatest + c);
    VSIE_CHECK_CUDA(cudaStreamCreateWithPriority(&h->chi_stream[c], cudaStreamNonBlocking, prio));
    VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_join[c], cudaEventDisableTiming));
  }
  VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
}

struct Streams {
  cudaStream_t main;
  cudaStream_t chi[3];
  bool parallel;
};

Streams make_streams(vsie_coupling_s* h, cudaStream_t main, bool parallel) {
  if (!parallel) return Streams{main, {main, main, main}, false};
  return Streams{main, {h->chi_stream[0], h->chi_stream[1], h->chi_stream[2]}, true};
}

void fork(vsie_coupling_s* h, const Streams& S) {
  if (!S.parallel) return;
  VSIE_CHECK_CUDA(cudaEventRecord(h->ev_fork, S.main));
  for (int c = 0; c < 3; ++c) VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.chi[c], h->ev_fork, 0));
}

void join(vsie_coupling_s* h, const Streams& S) {
  if (!S.parallel) return;
  for (int c = 0; c < 3; ++c) {
    VSIE_CHECK_CUDA(cudaEventRecord(h->ev_join[c], S.chi[c]));
    VSIE_CHECK_CUDA(cudaStreamWaitEvent(S.main, h->ev_join[c], 0));
  }
}

// ------------------------------------------------------------------ batched TMA passes (single RHS)
int64_t rsum3(const Ctx& X) { return X.R(0, 2) + X.R(1, 2) + X.R(2, 2); }

// the G4 pass over the three chi of one shard: y4 = G4 x (fwd) and / or
// z = sum_chi G4^T z3 (tr; written at zout, conj for op C) from ONE read of G4
void g4_pass(const Ctx& X, Shard& s, const cplx* x, cplx* zout, bool cj, cudaStream_t st) {
  vsie_coupling_s* h = X.h;
  if (s.mloc() == 0) {
    if (x) VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p, 0, 3 * X.r3stride * sizeof(cplx), st));
    return;
  }
  PairG4 p{};
  p.nbatch = 3;
  p.C = s.mloc();
  p.x = x ? x + s.cb : nullptr;
  p.z = zout;
  p.conj_z = cj;
  p.partials = X.partials(0);
  p.rstride = X.r3m;
  for (int c = 0; c < 3; ++c) {
    p.A[c] = s.G4[c].p;
    p.y4[c] = s.y4.p + c * X.r3stride;
    p.z3[c] = zout ? s.z3.p + c * X.r3stride : nullptr;
    p.R[c] = X.R(c, 2);
  }
  const int dirs = (x ? 1 : 0) + (zout ? 1 : 0);
  const char* name = dirs == 2 ? "pair_g4_tma" : x ? "fwd_g4_tma" : "adj_g4_tma";
  Scope sc(h, name, 16 * (rsum3(X) * (p.C + dirs) + dirs * p.C), 8 * dirs * rsum3(X) * p.C, st);
  VSIE_REQUIRE(launch_pair_g4(p, sm_count_dev(), st), VSIE_ERR_STATE, "G4 pass: unsupported shape");
}

// a G3 pass of one shard (k_seg_gemv on the row-blocked copy G3b): mode 1 Y3 = G3 y4,
// 2 z3 = G3^T W2, 3 both from one read; chi_only >= 0: that chi alone on a small ring (a
// chain's pass, leaving room on the SMs for the neighbouring chain's compute kernels)
void g3_pass(const Ctx& X, Shard& s, int mode, cudaStream_t st, int chi_only = -1) {
  vsie_coupling_s* h = X.h;
  const int64_t n3l = s.n3loc();
  SegGemv g{};
  g.nbatch = chi_only >= 0 ? 1 : 3;
  g.nsb = s.g3b_ns;
  g.partials = chi_only >= 0 ? X.partials(chi_only) : X.partials(0);
  g.rstride = X.r3m;
  int64_t bytes = 0;
  for (int i = 0; i < g.nbatch; ++i) {
    const int c = chi_only >= 0 ? chi_only : i;
    g.A[i] = s.G3b[c].p;
    g.R[i] = X.R(c, 1) * n3l;
    g.C[i] = X.R(c, 2);
    g.xparts[i] = 0;
    cplx* Y3 = s.Y3.p + c * X.r2m * n3l;
    cplx* W2 = s.W2.p + c * X.r2m * n3l;
    cplx* y4 = s.y4.p + c * X.r3stride;
    cplx* z3 = s.z3.p + c * X.r3stride;
    if (mode == 1) { g.x[i] = y4; g.y[i] = Y3; }
    if (mode == 2) { g.x[i] = W2; g.y[i] = z3; }
    if (mode == 3) { g.x[i] = y4; g.y[i] = Y3; g.xt[i] = W2; g.yt[i] = z3; }
    const int dirs = mode == 3 ? 2 : 1;
    bytes += 16 * (g.R[i] * g.C[i] + dirs * (g.R[i] + g.C[i]));
  }
  const char* name = mode == 3 ? "g3_seg_both" : mode == 1 ? (chi_only >= 0 ? "fwd_g3_seg_chi" : "fwd_g3_seg")
                                                            : "adj_g3_seg";
  Scope sc(h, name, bytes, mode == 3 ? bytes : bytes / 2, st);
  VSIE_REQUIRE(launch_seg_gemv_mode(g, mode, st, chi_only >= 0), VSIE_ERR_STATE, "G3 pass: unsupported shape");
}

// W2 = G2^T W1 for the three chi of one shard in one launch (k_g2t, no split-K partials);
// chi_only >= 0: that chi alone (inside its chain)
void g2t_pass(const Ctx& X, Shard& s, cudaStream_t st, int chi_only = -1) {
  vsie_coupling_s* h = X.h;
  const int n2 = h->grid.n[1];
  const int64_t n3l = s.n3loc();
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
    bytes += 16 * (X.R(c, 0) * n2 * X.R(c, 1) + X.R(c, 1) * n3l + X.R(c, 0) * n2 * n3l);
    fl += 8 * X.R(c, 0) * n2 * X.R(c, 1) * n3l;
  }
  Scope sc(h, chi_only >= 0 ? "adj_g2_g2t_chi" : "adj_g2_g2t", bytes, fl, st);
  launch_g2t(g, st);
}

bool tma_ok(vsie_coupling_s* h, const Ctx& X) {
  if (X.k != 1 || X.r3m > pair_g4_max_rank()) return false;
  for (Shard& s : h->shards) {
    if (s.n3loc() == 0 || s.mloc() == 0) return false;
    for (int c = 0; c < 3; ++c)
      if (!seg_gemv_supported(X.R(c, 1) * s.n3loc(), X.R(c, 2), s.g3b_ns)) return false;
  }
  return true;
}

// the forward's G3 pass per chi inside the chains (small ring) instead of one batched pass
// before them, so one chi's G2 / G1 work runs beside the next chi's G3 stream: measured
// cfg 2 (34 MB of G3 per chi) 0.1606 -> 0.1565 ms, cfg 4 (64 MB per chi) 0.4553 -> 0.4594
// ms; on when the largest per-chi G3 slice is <= 48 MB
bool fwd_chain_g3(vsie_coupling_s* h) {
  int64_t mx = 0;
  for (const Shard& s : h->shards)
    for (int c = 0; c < 3; ++c) mx = std::max<int64_t>(mx, 16LL * h->ranks[c][1] * s.n3loc() * h->ranks[c][2]);
  return mx <= (48LL << 20);
}

// the forward's steps after y4: Y3 (batched pass or per chi in the chains), G2 / G1 chains
void fwd_after_y4(const Ctx& X, cplx* y, const Streams& S) {
  vsie_coupling_s* h = X.h;
  const bool chain_g3 = fwd_chain_g3(h);
  if (!chain_g3)
    for (Shard& s : h->shards) g3_pass(X, s, 1, S.main);
  fork(h, S);
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) {
      if (chain_g3) g3_pass(X, s, 1, S.chi[c], c);
      fwd_tail(X, s, c, y, S.chi[c]);
    }
  }
  h->scope_chi = -1;
  join(h, S);
}

// the transpose's front up to W2.  Single RHS: the three chi's G1^T in ONE launch of the
// TMA-ring kernel (k_reduce_g1_tma: whole-stage bulk copies, consumers only compute; cfg 4
// 120 us for the three chi vs 151 us for three concurrent k_reduce_g1 chains),
// then one batched G2^T.  Block RHS: per-chi chains.  Measured and rejected
// (profiles/r02d/ab_last_session.json): per-chi TMA G1^T launches with chi c's G2^T beside
// chi c + 1's G1^T (cfg 4 0.439 vs 0.433 ms, cfg 2 0.165 vs 0.150), and an L2 prefetch of the
// head of G3 on a side stream under the FP64-bound G2^T (cfg 4 0.443, cfg 2 0.164-0.168).
void adj_front_w2(const Ctx& X, const cplx* u, bool cj, const Streams& S) {
  vsie_coupling_s* h = X.h;
  if (X.k == 1) {
    // single RHS: the three chi in ONE launch of the TMA-ring G1^T (k_reduce_g1_tma)
    for (Shard& s : h->shards) adj_g1_batched(X, s, u, cj, S.main);
    for (Shard& s : h->shards) g2t_pass(X, s, S.main);
    return;
  }
  fork(h, S);
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) adj_g1(X, s, c, u, cj, S.chi[c]);
  }
  h->scope_chi = -1;
  join(h, S);
  for (Shard& s : h->shards) g2t_pass(X, s, S.main);
}

// ------------------------------------------------------------------ the apply DAGs
// single RHS on the batched TMA passes
void apply_single_tma(Ctx X, const cplx* x, cplx* y, int op, const Streams& S) {
  vsie_coupling_s* h = X.h;
  if (op == VSIE_OP_N) {
    for (Shard& s : h->shards) g4_pass(X, s, x, nullptr, false, S.main);
    if (X.exchange()) combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
    fwd_after_y4(X, y, S);
    return;
  }
  const bool cj = op == VSIE_OP_C;
  X.ws = 3;   // the transpose's own workspaces: a forward apply may run beside it
  adj_front_w2(X, x, cj, S);
  for (Shard& s : h->shards) g3_pass(X, s, 2, S.main);
  if (X.exchange()) combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
  for (Shard& s : h->shards) g4_pass(X, s, nullptr, z_dest(h, s, y, 1), cj, S.main);
  gather_z(h, y, 1, S.main);
}

// per-chi kernel chains (block RHS; single-RHS shapes the TMA passes do not support)
void apply_chains(Ctx X, const cplx* x, cplx* y, int op, const Streams& S) {
  vsie_coupling_s* h = X.h;
  const bool exchange = X.exchange();
  fork(h, S);
  if (op == VSIE_OP_N) {
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) fwd_g4(X, s, c, x, S.chi[c]);
    }
    h->scope_chi = -1;
    if (exchange) {   // allreduce of the partial y4 (3 r3 values per RHS)
      join(h, S);
      combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
      fork(h, S);
    }
    for (int c = 0; c < 3; ++c) {
      h->scope_chi = c;
      for (Shard& s : h->shards) {
        if (s.n3loc() == 0) continue;
        fwd_g3(X, s, c, S.chi[c]);
        fwd_tail(X, s, c, y, S.chi[c]);
      }
    }
    h->scope_chi = -1;
    join(h, S);
    return;
  }
  const bool cj = op == VSIE_OP_C;
  X.ws = 3;
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) {
      if (s.n3loc() == 0) {
        VSIE_CHECK_CUDA(cudaMemsetAsync(s.z3.p + c * X.r3stride, 0, X.r3stride * sizeof(cplx), S.chi[c]));
        continue;
      }
      adj_g1(X, s, c, x, cj, S.chi[c]);
      adj_g2(X, s, c, S.chi[c]);
      adj_g3(X, s, c, S.chi[c]);
    }
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
  for (Shard& s : h->shards) adj_sum_chi(X, s, z_dest(h, s, y, X.k), z_ld(h), cj, S.main);
  gather_z(h, y, X.k, S.main);
}

void apply_dag(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, const Streams& S) {
  const Ctx X = make_ctx(h, nrhs);
  if (tma_ok(h, X))
    apply_single_tma(X, x, y, op, S);
  else
    apply_chains(X, x, y, op, S);
}

// bytes of the two large cores per shard: the pair schedule that reads the larger one once
bool g3_shared(vsie_coupling_s* h) {
  if (h->pair_sched == 1) return false;
  if (h->pair_sched == 2) return true;
  const Shard& s = h->shards[0];
  int64_t b3 = 0, b4 = 0;
  for (int c = 0; c < 3; ++c) {
    b3 += (int64_t)h->ranks[c][1] * s.n3loc() * h->ranks[c][2];
    b4 += (int64_t)h->ranks[c][2] * s.mloc();
  }
  return b3 > b4;
}

// The coupling pair of one GMRES matvec: y = Z x and z = Z^T u (Z^H u), single RHS.
void pair_dag(vsie_coupling_s* h, const cplx* x, cplx* y, const cplx* u, cplx* z, bool cj, const Streams& S) {
  const Ctx X = make_ctx(h, 1);
  const bool exchange = X.exchange();
  if (!g3_shared(h)) {
    // G4-shared: transpose front -> z3, ONE G4 pass for y4 and z, forward tail from y4
    adj_front_w2(X, u, cj, S);
    for (Shard& s : h->shards) g3_pass(X, s, 2, S.main);
    if (exchange) combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
    for (Shard& s : h->shards) g4_pass(X, s, x, z_dest(h, s, z, 1), cj, S.main);
    if (exchange) combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
    fwd_after_y4(X, y, S);
    gather_z(h, z, 1, S.main);
    return;
  }
  // G3-shared: the forward's G4 pass streams while the transpose's G1^T / G2^T chains
  // compute (per chi: chi c's G2^T runs beside chi c + 1's G1^T and the G4 stream).  Measured
  // against the alternatives at cfg 3 (profiles/r02c/g3s_schedules.json):
  // one batched TMA G1^T first and the G2^T beside the G4 stream 1.748 ms, fully serial
  // 1.737, the forward's G2 products first and the expansions beside the transpose's G4
  // stream 1.710-1.757, vs 1.683 ms for this one (a persistent G4 stream starves the
  // kernels beside it of SMs, so overlap only pays for short compute kernels)
  fork(h, S);
  for (Shard& s : h->shards) g4_pass(X, s, x, nullptr, false, S.main);
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) {
      adj_g1(X, s, c, u, cj, S.chi[c]);
      g2t_pass(X, s, S.chi[c], c);
    }
  }
  h->scope_chi = -1;
  join(h, S);
  if (exchange) combine_r3(h, &Shard::y4, 3 * X.r3stride, S.main);
  // ONE pass over G3: Y3 = G3 y4 and z3 = G3^T W2
  for (Shard& s : h->shards) g3_pass(X, s, 3, S.main);
  if (exchange) combine_r3(h, &Shard::z3, 3 * X.r3stride, S.main);
  // the transpose's G4 pass streams while the forward's G2 / G1 chains compute
  fork(h, S);
  for (Shard& s : h->shards) g4_pass(X, s, nullptr, z_dest(h, s, z, 1), cj, S.main);
  for (int c = 0; c < 3; ++c) {
    h->scope_chi = c;
    for (Shard& s : h->shards) fwd_tail(X, s, c, y, S.chi[c]);
  }
  h->scope_chi = -1;
  join(h, S);
  gather_z(h, z, 1, S.main);
}

bool graphs_enabled(vsie_coupling_s* h) {
  // multi-process handles run eagerly: their collectives may synchronise with the host
  // (the single-GPU IPC communicator) and NCCL inside captured graphs is not exercised here
  return h->use_graphs && !h->timing && !h->comm;
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
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
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
  if (h->timing && !h->comm) {
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
    // eager; per-kernel timing of a multi-process handle serialises on the caller's stream
    Streams S = make_streams(h, st, !h->timing);
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
  if (!tma_ok(h, make_ctx(h, 1))) {   // shapes the fused passes do not support: two applies
    apply(h, x, y, VSIE_OP_N, 1, st);
    apply(h, u, z, adj_op, 1, st);
    return;
  }
  run_dag(h, 100 + adj_op, 1, x, y, u, z, st,
          [&](const Streams& S) { pair_dag(h, x, y, u, z, adj_op == VSIE_OP_C, S); });
}

int pair_schedule(vsie_coupling_s* h) { return g3_shared(h) ? 2 : 1; }

}  // namespace vsie
