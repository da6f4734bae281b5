// Handle setup, slab partition (SURVEY §8e design iii) and the TT apply
// orchestration (forward Eq. 17, transpose Eqs. 18-19) over the kernels of
// ttapply.cu / linalg.cu.
#include "handle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace vsie {

namespace {

// ------------------------------------------------------------------ small kernels
// TT value at (row, col): chain product G1[i1,:] G2[:,i2,:] G3[:,i3,:] G4[:,n] (Eq. 9).
struct EvalCores {
  const cplx* G[3][4];
  int r[3][3];
};
__global__ void k_tt_eval(EvalCores c, int n1, int n2, int n3, int64_t nv, const int64_t* __restrict__ idx,
                          int64_t count, cplx* __restrict__ out) {
  extern __shared__ cplx sv[];
  __shared__ double red[2][32];
  for (int64_t e = blockIdx.x; e < count; e += gridDim.x) {
    const int64_t row = idx[2 * e], n = idx[2 * e + 1];
    const int chi = (int)(row / nv);
    const int64_t v = row - chi * nv;
    const int i1 = (int)(v % n1), i2 = (int)((v / n1) % n2), i3 = (int)(v / ((int64_t)n1 * n2));
    const int r1 = c.r[chi][0], r2 = c.r[chi][1], r3 = c.r[chi][2];
    cplx* v1 = sv;
    cplx* v2 = sv + r1;
    cplx* v3 = v2 + r2;
    __syncthreads();
    for (int a = threadIdx.x; a < r1; a += blockDim.x) v1[a] = c.G[chi][0][i1 + (int64_t)n1 * a];
    __syncthreads();
    for (int b = threadIdx.x; b < r2; b += blockDim.x) {
      cplx s = cmk(0, 0);
      for (int a = 0; a < r1; ++a) cfma(s, v1[a], c.G[chi][1][a + (int64_t)r1 * (i2 + (int64_t)n2 * b)]);
      v2[b] = s;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < r3; b += blockDim.x) {
      cplx s = cmk(0, 0);
      for (int a = 0; a < r2; ++a) cfma(s, v2[a], c.G[chi][2][a + (int64_t)r2 * (i3 + (int64_t)n3 * b)]);
      v3[b] = s;
    }
    __syncthreads();
    cplx s = cmk(0, 0);
    for (int a = threadIdx.x; a < r3; a += blockDim.x) cfma(s, v3[a], c.G[chi][3][a + (int64_t)r3 * n]);
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { red[0][w] = s.x; red[1][w] = s.y; }
    __syncthreads();
    if (threadIdx.x == 0) {
      cplx t = cmk(0, 0);
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { t.x += red[0][q]; t.y += red[1][q]; }
      out[e] = t;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ setup
void handle_init_geometry(vsie_coupling_s* h, const vsie_grid* grid, const vsie_mesh* meshes, int n_meshes,
                          double freq, const vsie_build_opts* o) {
  VSIE_REQUIRE(freq > 0 && std::isfinite(freq), VSIE_ERR_ARG, "freq must be > 0");
  h->grid = make_grid(grid);
  VSIE_REQUIRE(o->quad_rule == 0 || o->quad_rule == 1, VSIE_ERR_ARG, "quad_rule must be 0 or 1");
  h->quad_rule = o->quad_rule;
  h->sources = build_sources(meshes, n_meshes, h->grid, h->quad_rule == 1 ? 1 : 3);
  h->m = h->sources.m;
  {
    uint64_t f = 1469598103934665603ull;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(h->sources.table.data());
    for (size_t i = 0; i < h->sources.table.size() * sizeof(double); ++i) f = (f ^ b[i]) * 1099511628211ull;
    h->src_hash = f;
  }
  const double c0 = 299792458.0;
  h->k0 = 2.0 * M_PI * freq / c0;
  h->scale_re = o->scale_re;
  h->scale_im = o->scale_im;
  h->rank = o->rank;
  h->world = o->world;
  h->loopback = o->loopback;
  h->nrhs_max = o->nrhs_max;
  VSIE_REQUIRE(h->world >= 1 && h->rank >= 0 && h->rank < h->world, VSIE_ERR_ARG, "bad rank/world");
  VSIE_REQUIRE(h->nrhs_max >= 1 && h->nrhs_max <= 4096, VSIE_ERR_ARG, "bad nrhs_max");
  VSIE_REQUIRE(h->grid.n[2] >= h->world, VSIE_ERR_ARG, "n3 must be >= world for the i3 slab partition");
  if (o->device >= 0) VSIE_CHECK_CUDA(cudaSetDevice(o->device));
  VSIE_CHECK_CUDA(cudaGetDevice(&h->device));
  h->d_src.alloc(h->sources.table.size());
  VSIE_CHECK_CUDA(cudaMemcpy(h->d_src.p, h->sources.table.data(), h->sources.table.size() * sizeof(double),
                             cudaMemcpyHostToDevice));
  EntryGeom& g = h->eg;
  g.n1 = h->grid.n[0];
  g.n2 = h->grid.n[1];
  g.n3 = h->grid.n[2];
  g.ox = h->grid.origin[0];
  g.oy = h->grid.origin[1];
  g.oz = h->grid.origin[2];
  g.hx = h->grid.h[0];
  g.hy = h->grid.h[1];
  g.hz = h->grid.h[2];
  const double s3 = 2.0 * std::sqrt(3.0);
  g.dx = g.hx / s3;
  g.dy = g.hy / s3;
  g.dz = g.hz / s3;
  // quad_rule 1 (P:287 far block): one node at the voxel centre with the whole voxel weight,
  // one centroid per triangle; otherwise 2 x 2 x 2 Gauss nodes x the 3-point triangle rule
  g.nodes = h->quad_rule == 1 ? 1 : 8;
  g.nsrc = h->quad_rule == 1 ? 2 : 6;
  g.w = g.hx * g.hy * g.hz / (g.nodes == 1 ? 1.0 : 8.0);
  // node p = (sigma1, sigma2, sigma3) with bit l-1 of p set for +h_l / (2 sqrt 3): the linear
  // PWL test function (r_p - c)_l / h_l is +-1 / (2 sqrt 3) there (DESIGN.md R-PWL)
  h->test_moment = o->test_moment;
  VSIE_REQUIRE(h->test_moment >= 0 && h->test_moment <= 3, VSIE_ERR_ARG, "test_moment must be 0..3");
  const double inv4pi = 0.079577471545947667884441881686257181;   // 1/(4 pi)
  for (int p = 0; p < 8; ++p) {
    const int l = h->test_moment;
    g.pw[p] = l == 0 ? inv4pi : (((p >> (l - 1)) & 1) ? inv4pi / s3 : -inv4pi / s3);
    if (g.nodes == 1 && l != 0) g.pw[p] = 0.0;   // the linear test function vanishes at the centre
  }
  g.k0 = h->k0;
  g.inv_k0 = 1.0 / h->k0;
  // |delta| <= k0 |d|: the order-7 phase polynomial is exact to < 1e-19 while k0 |d| <= 0.03
  g.taylor = h->k0 * std::sqrt(g.dx * g.dx + g.dy * g.dy + g.dz * g.dz) <= 0.03 ? 1 : 0;
  g.scale_re = h->scale_re;
  g.scale_im = h->scale_im;
  g.src = h->d_src.p;
  g.m = h->m;
  g.nv = h->grid.nv();
  if (h->world > 1 && !h->loopback) {
    if (o->ipc_name) {
      VSIE_REQUIRE(std::strlen(o->ipc_name) > 0 && std::strlen(o->ipc_name) <= 200, VSIE_ERR_ARG, "bad ipc_name");
      h->comm.reset(make_ipc_comm(o->ipc_name, h->rank, h->world));
    } else {
      VSIE_REQUIRE(o->nccl_unique_id != nullptr, VSIE_ERR_ARG, "world > 1 needs nccl_unique_id or ipc_name");
      h->comm.reset(make_nccl_comm(o->nccl_unique_id, h->rank, h->world));
    }
  }
  handle_partition(h);
}

void slab_partition(int n3, int64_t m, int world, int rank, int slab[2], int64_t cols[2]) {
  const int64_t mp = ceil_div(m, world);
  slab[0] = (int)((int64_t)n3 * rank / world);
  slab[1] = (int)((int64_t)n3 * (rank + 1) / world);
  cols[0] = std::min(m, mp * rank);
  cols[1] = std::min(m, mp * (rank + 1));
}

void handle_partition(vsie_coupling_s* h) {
  const int P = h->world;
  h->shards.clear();
  const int first = h->loopback ? 0 : h->rank;
  const int last = h->loopback ? P : h->rank + 1;
  h->shards.resize(last - first);
  for (int p = first; p < last; ++p) {
    Shard& s = h->shards[p - first];
    int sl[2];
    int64_t cl[2];
    slab_partition(h->grid.n[2], h->m, P, p, sl, cl);
    s.i3b = sl[0];
    s.i3e = sl[1];
    s.cb = cl[0];
    s.ce = cl[1];
  }
}

void handle_alloc_workspace(vsie_coupling_s* h) {
  const int k = h->nrhs_max;
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  int r1m = 1, r2m = 1, r3m = 1;
  for (int c = 0; c < 3; ++c) {
    r1m = std::max(r1m, h->ranks[c][0]);
    r2m = std::max(r2m, h->ranks[c][1]);
    r3m = std::max(r3m, h->ranks[c][2]);
  }
  // row-blocked copies of the G3 slices (k_seg_gemv)
  const int nsb = sm_count_dev();
  for (Shard& s : h->shards) {
    s.g3b_ns = nsb;
    for (int c = 0; c < 3; ++c) {
      const int64_t R = (int64_t)h->ranks[c][1] * s.n3loc(), C = h->ranks[c][2];
      s.G3b[c].alloc((size_t)std::max<int64_t>(1, R * C));
      if (R == 0) continue;
      for (int q = 0; q < nsb; ++q) {
        const int64_t r0 = R * q / nsb, L = R * (q + 1) / nsb - r0;
        if (L == 0) continue;
        VSIE_CHECK_CUDA(cudaMemcpy2D(s.G3b[c].p + C * r0, L * sizeof(cplx), s.G3[c].p + r0, R * sizeof(cplx),
                                     L * sizeof(cplx), C, cudaMemcpyDeviceToDevice));
      }
    }
  }
  for (Shard& s : h->shards) {
    const int64_t n3l = std::max(1, s.n3loc());
    s.y4.alloc(3 * (int64_t)r3m * k);
    s.z3.alloc(3 * (int64_t)r3m * k);
    s.Y3.alloc(3 * (int64_t)r2m * n3l * k);
    s.W2.alloc(3 * (int64_t)r2m * n3l * k);
    s.Y2.alloc(3 * (int64_t)r1m * n2 * n3l * k);
    s.W1.alloc(3 * (int64_t)r1m * n2 * n3l * k);
  }
  (void)n1;
  // per-chi split-K partials of the GEMVs (the launchers lower the split to fit) and the
  // per-CTA partials of the batched TMA passes ([chi][CTA][r3max] from partials(0), so a
  // region of three chi holds 3 nsm r3max): the three chi chains of an apply run concurrently
  h->partials_per_chi = std::max<int64_t>(400000, (int64_t)nsb * r3m);
  h->partials.alloc((size_t)6 * h->partials_per_chi);   // [fwd chi 0..2][adj chi 0..2]
  int64_t wsz = 64 * std::max<int64_t>((int64_t)r2m * std::max(1, h->shards[0].n3loc()) * k, (int64_t)r3m * k);
  h->zgemm_ws_per_chi = std::min<int64_t>(wsz, (int64_t)16 << 20);
  h->zgemm_ws.alloc((size_t)6 * h->zgemm_ws_per_chi);
  // per-chi partial surface vectors of the transpose (z_chi = G4_chi^T z3_chi)
  int64_t mloc_max = 1;
  for (Shard& s : h->shards) mloc_max = std::max<int64_t>(mloc_max, s.mloc());
  for (Shard& s : h->shards) s.zpart.alloc((size_t)3 * mloc_max * k);
  apply_reset_graphs(h);
  if (h->comm) {
    const int64_t mp = ceil_div(h->m, h->world);
    h->gather_buf.alloc((size_t)(h->world + 1) * mp * k);
  }
}

static void set_cores_common(vsie_coupling_s* h, int chi, const int r[3], const cplx* const src[4],
                             cudaMemcpyKind kind) {
  VSIE_REQUIRE(chi >= 0 && chi < 3, VSIE_ERR_ARG, "chi out of range");
  for (int k = 0; k < 3; ++k) VSIE_REQUIRE(r[k] >= 1 && r[k] <= 65536, VSIE_ERR_ARG, "rank out of range");
  for (int k = 0; k < 4; ++k) VSIE_REQUIRE(src[k] != nullptr, VSIE_ERR_ARG, "core pointer is NULL");
  const int n1 = h->grid.n[0], n2 = h->grid.n[1], n3 = h->grid.n[2];
  const int r1 = r[0], r2 = r[1], r3 = r[2];
  h->ranks[chi][0] = r1;
  h->ranks[chi][1] = r2;
  h->ranks[chi][2] = r3;
  h->G1[chi].alloc((size_t)n1 * r1);
  h->G2[chi].alloc((size_t)r1 * n2 * r2);
  const cudaMemcpyKind k1 = kind;
  VSIE_CHECK_CUDA(cudaMemcpy(h->G1[chi].p, src[0], h->G1[chi].bytes(), k1));
  VSIE_CHECK_CUDA(cudaMemcpy(h->G2[chi].p, src[1], h->G2[chi].bytes(), k1));
  for (Shard& s : h->shards) {
    const int n3l = s.n3loc();
    s.G3[chi].alloc((size_t)r2 * std::max(n3l, 1) * r3);
    // G3(a2, i3, a3) at a2 + r2 (i3 + n3 a3): the owned slice is, per a3, a
    // contiguous run of r2 * n3l elements starting at r2 * (i3b + n3 a3).
    if (n3l > 0)
      VSIE_CHECK_CUDA(cudaMemcpy2D(s.G3[chi].p, (size_t)r2 * n3l * sizeof(cplx), src[2] + (size_t)r2 * s.i3b,
                                   (size_t)r2 * n3 * sizeof(cplx), (size_t)r2 * n3l * sizeof(cplx), r3, k1));
    s.G4[chi].alloc((size_t)r3 * std::max<int64_t>(s.mloc(), 1));
    if (s.mloc() > 0)
      VSIE_CHECK_CUDA(cudaMemcpy(s.G4[chi].p, src[3] + (size_t)r3 * s.cb, (size_t)r3 * s.mloc() * sizeof(cplx), k1));
  }
  (void)n3;
}

void handle_set_cores_host(vsie_coupling_s* h, int chi, const int r[3], const cplx* const host[4]) {
  set_cores_common(h, chi, r, host, cudaMemcpyHostToDevice);
}
void handle_set_cores_device(vsie_coupling_s* h, int chi, const int r[3], const cplx* const dev[4]) {
  set_cores_common(h, chi, r, dev, cudaMemcpyDeviceToDevice);
}

void tt_eval(vsie_coupling_s* h, const int64_t* idx, int64_t count, cplx* out, cudaStream_t st) {
  VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
  VSIE_REQUIRE(h->world == 1 && h->shards.size() == 1, VSIE_ERR_STATE, "tt_eval needs world == 1");
  if (count <= 0) return;
  EvalCores c{};
  int rmax = 1;
  for (int q = 0; q < 3; ++q) {
    c.G[q][0] = h->G1[q].p;
    c.G[q][1] = h->G2[q].p;
    c.G[q][2] = h->shards[0].G3[q].p;
    c.G[q][3] = h->shards[0].G4[q].p;
    for (int j = 0; j < 3; ++j) c.r[q][j] = h->ranks[q][j];
    rmax = std::max(rmax, h->ranks[q][0] + h->ranks[q][1] + h->ranks[q][2]);
  }
  const size_t smem = (size_t)rmax * sizeof(cplx);
  VSIE_REQUIRE(smem <= 200 * 1024, VSIE_ERR_ARG, "ranks too large for tt_eval");
  VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_tt_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int blocks = (int)std::min<int64_t>(count, 148 * 16);
  k_tt_eval<<<blocks, 128, smem, st>>>(c, h->grid.n[0], h->grid.n[1], h->grid.n[2], h->grid.nv(), idx, count, out);
  VSIE_CHECK_LAUNCH();
}

void launch_tt_eval(const cplx* const G[4], const int r[3], const int n[3], int64_t m, int chi_sel,
                    const int64_t* idx, int64_t count, int64_t nv, cplx* out, cudaStream_t st) {
  (void)m;
  (void)chi_sel;
  if (count <= 0) return;
  EvalCores c{};
  for (int q = 0; q < 3; ++q) {
    for (int k = 0; k < 4; ++k) c.G[q][k] = G[k];
    for (int j = 0; j < 3; ++j) c.r[q][j] = r[j];
  }
  const size_t smem = (size_t)(r[0] + r[1] + r[2]) * sizeof(cplx);
  VSIE_REQUIRE(smem <= 200 * 1024, VSIE_ERR_ARG, "ranks too large for tt_eval");
  static bool configured = false;
  if (!configured) {
    VSIE_CHECK_CUDA(cudaFuncSetAttribute(k_tt_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  const int blocks = (int)std::min<int64_t>(count, 148 * 16);
  k_tt_eval<<<blocks, 128, smem, st>>>(c, n[0], n[1], n[2], nv, idx, count, out);
  VSIE_CHECK_LAUNCH();
}

}  // namespace vsie

vsie_coupling_s::~vsie_coupling_s() {
  for (auto& t : pending) {
    cudaEventDestroy(t.e0);
    cudaEventDestroy(t.e1);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (io_stream) cudaStreamDestroy(io_stream);
  if (io_stream2) cudaStreamDestroy(io_stream2);
  if (pwl_stream) cudaStreamDestroy(pwl_stream);
  if (pwl_ev_fork) cudaEventDestroy(pwl_ev_fork);
  if (pwl_ev_done) cudaEventDestroy(pwl_ev_done);
  vsie::apply_destroy(this);
}
