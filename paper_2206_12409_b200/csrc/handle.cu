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

// copy a (rows x cols) column-major block with source ld / dest ld
void copy2d(cplx* dst, int64_t ldd, const cplx* src, int64_t lds, int64_t rows, int64_t cols,
            cudaMemcpyKind kind, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  VSIE_CHECK_CUDA(cudaMemcpy2DAsync(dst, ldd * sizeof(cplx), src, lds * sizeof(cplx), rows * sizeof(cplx),
                                    cols, kind, st));
}

}  // namespace

// ------------------------------------------------------------------ timing scopes
struct Scope {
  vsie_coupling_s* h;
  size_t slot;
  bool on;
  Scope(vsie_coupling_s* hh, const char* name, int64_t bytes, int64_t flops, cudaStream_t st) : h(hh), on(hh->timing) {
    if (!on) return;
    Timed t;
    t.name = name;
    t.bytes = bytes;
    t.flops = flops;
    if (h->event_pool.size() < 2) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        VSIE_CHECK_CUDA(cudaEventCreate(&e));
        h->event_pool.push_back(e);
      }
    }
    t.e0 = h->event_pool.back(); h->event_pool.pop_back();
    t.e1 = h->event_pool.back(); h->event_pool.pop_back();
    VSIE_CHECK_CUDA(cudaEventRecord(t.e0, st));
    h->pending.push_back(t);
    slot = h->pending.size() - 1;
    stream = st;
  }
  cudaStream_t stream = nullptr;
  ~Scope() {
    if (on) cudaEventRecord(h->pending[slot].e1, stream);
  }
};

// ------------------------------------------------------------------ setup
void handle_init_geometry(vsie_coupling_s* h, const vsie_grid* grid, const vsie_mesh* meshes, int n_meshes,
                          double freq, const vsie_build_opts* o) {
  VSIE_REQUIRE(freq > 0 && std::isfinite(freq), VSIE_ERR_ARG, "freq must be > 0");
  h->grid = make_grid(grid);
  h->sources = build_sources(meshes, n_meshes, h->grid);
  h->m = h->sources.m;
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
  g.w = g.hx * g.hy * g.hz / 8.0;
  g.k0 = h->k0;
  g.inv_k0 = 1.0 / h->k0;
  g.scale_re = h->scale_re;
  g.scale_im = h->scale_im;
  g.src = h->d_src.p;
  g.m = h->m;
  g.nv = h->grid.nv();
  if (h->world > 1 && !h->loopback) {
    VSIE_REQUIRE(o->nccl_unique_id != nullptr, VSIE_ERR_ARG, "world > 1 needs nccl_unique_id");
    h->comm.reset(make_nccl_comm(o->nccl_unique_id, h->rank, h->world));
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
  int64_t rmax_gemv = 1;
  for (Shard& s : h->shards) {
    const int64_t n3l = std::max(1, s.n3loc());
    s.y4.alloc(3 * (int64_t)r3m * k);
    s.z3.alloc(3 * (int64_t)r3m * k);
    s.Y3.alloc(3 * (int64_t)r2m * n3l * k);
    s.W2.alloc(3 * (int64_t)r2m * n3l * k);
    s.Y2.alloc(3 * (int64_t)r1m * n2 * n3l * k);
    rmax_gemv = std::max(rmax_gemv, (int64_t)r2m * n3l);
  }
  (void)n1;
  (void)rmax_gemv;
  // split-K partials: the launchers cap splits so that nsplit * rows <= 888/3 * 256
  // (gemv_n) and nsplit * cols <= 888/3 * 32 (gemv_t) per batch
  h->partials.alloc((size_t)3 * 320000);
  h->counters.alloc(3 * 8192);
  VSIE_CHECK_CUDA(cudaMemset(h->counters.p, 0, h->counters.bytes()));
  // split-K workspace of the ZGEMMs (launch_zgemm lowers the split to fit)
  int64_t wsz = 3 * 64 * std::max<int64_t>((int64_t)r2m * std::max(1, h->shards[0].n3loc()) * k, (int64_t)r3m * k);
  h->zgemm_ws.alloc((size_t)std::min<int64_t>(wsz, (int64_t)32 << 20));
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

// ------------------------------------------------------------------ apply
namespace {

struct IoLayout {
  // voxel-side vector of this handle: base pointer of the whole buffer the
  // caller passed, offset of chi block and of this shard's planes, ld per RHS
  int64_t chi_stride;   // elements between chi blocks
  int64_t ld;           // elements between RHS columns
  bool global;          // true: buffer is the global 3 n_v vector (world 1 / loopback)
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

void combine_r3(vsie_coupling_s* h, DevBuf<cplx> Shard::*buf, int64_t n, cudaStream_t st) {
  // sum the per-shard partial vectors (3 * r3max * nrhs) across ranks/shards
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

}  // namespace

static void apply_impl(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st);

void apply(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st) {
  const int64_t before = launch_counter();
  apply_impl(h, x, y, op, nrhs, st);
  h->apply_launches += launch_counter() - before;
  h->apply_calls += 1;
}

static void apply_impl(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st) {
  VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "bad op");
  VSIE_REQUIRE(nrhs >= 1 && nrhs <= h->nrhs_max, VSIE_ERR_ARG, "nrhs out of range");
  VSIE_REQUIRE(x != nullptr && y != nullptr, VSIE_ERR_ARG, "x / y is NULL");
  const int n1 = h->grid.n[0], n2 = h->grid.n[1];
  const int64_t m = h->m;
  const int k = nrhs;
  int r1m = 1, r2m = 1, r3m = 1;
  for (int c = 0; c < 3; ++c) {
    r1m = std::max(r1m, h->ranks[c][0]);
    r2m = std::max(r2m, h->ranks[c][1]);
    r3m = std::max(r3m, h->ranks[c][2]);
  }
  // per-chi strides of the workspaces (sized with the max rank over chi)
  const int64_t r3stride = (int64_t)r3m * k;
  const IoLayout L = voxel_layout(h);
  const int max_splits = 256;
  auto R = [&](int c, int j) { return (int64_t)h->ranks[c][j]; };

  if (op == VSIE_OP_N) {
    // ---- step 1: y4 = G4[:, owned] x[owned], partial per shard
    for (Shard& s : h->shards) {
      if (k == 1) {
        GemvN g{};
        g.nbatch = 3;
        int64_t bytes = 16 * s.mloc();
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G4[c].p;
          g.x[c] = x + s.cb;
          g.y[c] = s.y4.p + c * r3stride;
          g.R[c] = R(c, 2);
          g.C[c] = s.mloc();
          bytes += 16 * R(c, 2) * s.mloc();
        }
        Scope sc(h, "fwd_g4_gemv", bytes, 8 * (bytes / 16), st);
        if (s.mloc() > 0)
          launch_gemv_n(g, h->partials.p, (int64_t)h->partials.n, max_splits, st);
        else
          VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p, 0, s.y4.bytes(), st));
      } else {
        Zgemm z{};
        z.nbatch = 3;
        for (int c = 0; c < 3; ++c) {
          z.M[c] = R(c, 2); z.N[c] = k; z.K[c] = s.mloc();
          z.A[c] = s.G4[c].p; z.lda[c] = R(c, 2);
          z.B[c] = x + s.cb; z.ldb[c] = m;
          z.C[c] = s.y4.p + c * r3stride; z.ldc[c] = R(c, 2);
        }
        Scope sc(h, "fwd_g4_zgemm", 0, 0, st);
        if (s.mloc() > 0)
          launch_zgemm(z, h->zgemm_ws.p, h->zgemm_ws.n, st);
        else
          VSIE_CHECK_CUDA(cudaMemsetAsync(s.y4.p, 0, s.y4.bytes(), st));
      }
    }
    // ---- combine partial y4 across ranks (allreduce of 3 r3 values)
    combine_r3(h, &Shard::y4, 3 * r3stride, st);
    for (Shard& s : h->shards) {
      const int64_t n3l = s.n3loc();
      if (n3l == 0) continue;
      // ---- step 2: Y3 = G3[:, owned i3, :] y4
      if (k == 1) {
        GemvN g{};
        g.nbatch = 3;
        int64_t bytes = 0;
        for (int c = 0; c < 3; ++c) {
          g.A[c] = s.G3[c].p;
          g.x[c] = s.y4.p + c * r3stride;
          g.y[c] = s.Y3.p + c * r2m * n3l;
          g.R[c] = R(c, 1) * n3l;
          g.C[c] = R(c, 2);
          bytes += 16 * (R(c, 1) * n3l * R(c, 2) + R(c, 1) * n3l + R(c, 2));
        }
        Scope sc(h, "fwd_g3_gemv", bytes, 8 * (bytes / 16), st);
        launch_gemv_n(g, h->partials.p, (int64_t)h->partials.n, max_splits, st);
      } else {
        Zgemm z{};
        z.nbatch = 3;
        for (int c = 0; c < 3; ++c) {
          z.M[c] = R(c, 1) * n3l; z.N[c] = k; z.K[c] = R(c, 2);
          z.A[c] = s.G3[c].p; z.lda[c] = R(c, 1) * n3l;
          z.B[c] = s.y4.p + c * r3stride; z.ldb[c] = R(c, 2);
          z.C[c] = s.Y3.p + c * r2m * n3l * k; z.ldc[c] = R(c, 1) * n3l;
        }
        Scope sc(h, "fwd_g3_zgemm", 0, 0, st);
        launch_zgemm(z, h->zgemm_ws.p, h->zgemm_ws.n, st);
      }
      // ---- step 3: Y2 = G2 Y3  ((r1 n2) x r2 times r2 x (n3l k))
      {
        Zgemm z{};
        z.nbatch = 3;
        int64_t bytes = 0, flops = 0;
        for (int c = 0; c < 3; ++c) {
          z.M[c] = R(c, 0) * n2; z.N[c] = n3l * k; z.K[c] = R(c, 1);
          z.A[c] = h->G2[c].p; z.lda[c] = R(c, 0) * n2;
          z.B[c] = s.Y3.p + c * r2m * n3l * k; z.ldb[c] = R(c, 1);
          z.C[c] = s.Y2.p + c * r1m * n2 * n3l * k; z.ldc[c] = R(c, 0) * n2;
          bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l * k + R(c, 0) * n2 * n3l * k);
          flops += 8 * R(c, 0) * n2 * R(c, 1) * n3l * k;
        }
        Scope sc(h, "fwd_g2_zgemm", bytes, flops, st);
        launch_zgemm_dmma(z, h->zgemm_ws.p, h->zgemm_ws.n, st);
      }
      // ---- step 4: y = G1 Y2 into the voxel slab
      {
        ExpandArgs e{};
        e.nbatch = 3;
        e.n1 = n1;
        e.ncol = (int64_t)n2 * n3l * k;
        e.cols_per_rhs = (int64_t)n2 * n3l;
        e.ld_rhs = L.ld;
        int64_t bytes = 0, flops = 0;
        const int64_t off = shard_voxel_offset(h, s, L);
        for (int c = 0; c < 3; ++c) {
          e.G1[c] = h->G1[c].p;
          e.Y2[c] = s.Y2.p + c * r1m * n2 * n3l * k;
          e.y[c] = y + c * L.chi_stride + off;
          e.r1[c] = h->ranks[c][0];
          bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k);
          flops += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l * k;
        }
        Scope sc(h, "fwd_g1_expand", bytes, flops, st);
        launch_expand_g1(e, st);
      }
    }
    return;
  }

  // ================= transpose / conjugate transpose
  const bool cj = op == VSIE_OP_C;
  for (Shard& s : h->shards) {
    const int64_t n3l = s.n3loc();
    if (n3l == 0) {
      VSIE_CHECK_CUDA(cudaMemsetAsync(s.z3.p, 0, s.z3.bytes(), st));
      continue;
    }
    // ---- W1 = G1^T u
    {
      ReduceArgs r{};
      r.nbatch = 3;
      r.n1 = n1;
      r.ncol = (int64_t)n2 * n3l * k;
      r.cols_per_rhs = (int64_t)n2 * n3l;
      r.ld_rhs = L.ld;
      r.conj_u = cj;
      const int64_t off = shard_voxel_offset(h, s, L);
      int64_t bytes = 0, flops = 0;
      for (int c = 0; c < 3; ++c) {
        r.G1[c] = h->G1[c].p;
        r.u[c] = x + c * L.chi_stride + off;
        r.W1[c] = s.Y2.p + c * r1m * n2 * n3l * k;
        r.r1[c] = h->ranks[c][0];
        bytes += 16 * ((int64_t)n1 * R(c, 0) + R(c, 0) * n2 * n3l * k + (int64_t)n1 * n2 * n3l * k);
        flops += 8 * (int64_t)n1 * R(c, 0) * n2 * n3l * k;
      }
      Scope sc(h, "adj_g1_reduce", bytes, flops, st);
      launch_reduce_g1(r, st);
    }
    // ---- W2 = G2^T W1
    {
      Zgemm z{};
      z.nbatch = 3;
      z.ta = kT;
      int64_t bytes = 0, flops = 0;
      for (int c = 0; c < 3; ++c) {
        z.M[c] = R(c, 1); z.N[c] = n3l * k; z.K[c] = R(c, 0) * n2;
        z.A[c] = h->G2[c].p; z.lda[c] = R(c, 0) * n2;
        z.B[c] = s.Y2.p + c * r1m * n2 * n3l * k; z.ldb[c] = R(c, 0) * n2;
        z.C[c] = s.W2.p + c * r2m * n3l * k; z.ldc[c] = R(c, 1);
        bytes += 16 * (R(c, 0) * n2 * R(c, 1) + R(c, 1) * n3l * k + R(c, 0) * n2 * n3l * k);
        flops += 8 * R(c, 0) * n2 * R(c, 1) * n3l * k;
      }
      Scope sc(h, "adj_g2_zgemm", bytes, flops, st);
      launch_zgemm_dmma(z, h->zgemm_ws.p, h->zgemm_ws.n, st);
    }
    // ---- z3 = G3^T W2, partial over the owned planes
    if (k == 1) {
      GemvT g{};
      g.nbatch = 3;
      int64_t bytes = 0;
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G3[c].p;
        g.x[c] = s.W2.p + c * r2m * n3l;
        g.y[c] = s.z3.p + c * r3stride;
        g.R[c] = R(c, 1) * n3l;
        g.C[c] = R(c, 2);
        bytes += 16 * (R(c, 1) * n3l * R(c, 2) + R(c, 1) * n3l + R(c, 2));
      }
      Scope sc(h, "adj_g3_gemv", bytes, 8 * (bytes / 16), st);
      launch_gemv_t(g, h->partials.p, (int64_t)h->partials.n, max_splits, st);
    } else {
      Zgemm z{};
      z.nbatch = 3;
      z.ta = kT;
      for (int c = 0; c < 3; ++c) {
        z.M[c] = R(c, 2); z.N[c] = k; z.K[c] = R(c, 1) * n3l;
        z.A[c] = s.G3[c].p; z.lda[c] = R(c, 1) * n3l;
        z.B[c] = s.W2.p + c * r2m * n3l * k; z.ldb[c] = R(c, 1) * n3l;
        z.C[c] = s.z3.p + c * r3stride; z.ldc[c] = R(c, 2);
      }
      Scope sc(h, "adj_g3_zgemm", 0, 0, st);
      launch_zgemm(z, h->zgemm_ws.p, h->zgemm_ws.n, st);
    }
  }
  // ---- combine z3 across ranks (allreduce of 3 r3 values)
  combine_r3(h, &Shard::z3, 3 * r3stride, st);
  // ---- z[owned] = sum_chi G4[:, owned]^T z3  (Eq. 18 sum over chi)
  const int64_t mp = ceil_div(m, h->world);
  for (Shard& s : h->shards) {
    if (s.mloc() == 0) continue;
    cplx* zout;
    int64_t ldz;
    if (h->comm) {
      zout = h->gather_buf.p + (int64_t)h->world * mp * k;  // local segment staging [mp x k]
      ldz = mp;
    } else {
      zout = y + s.cb;
      ldz = m;
    }
    if (k == 1) {
      GemvT g{};
      g.nbatch = 3;
      g.sum_batch = true;
      g.conj_out = cj;
      int64_t bytes = 16 * s.mloc();
      for (int c = 0; c < 3; ++c) {
        g.A[c] = s.G4[c].p;
        g.x[c] = s.z3.p + c * r3stride;
        g.y[c] = zout;
        g.R[c] = R(c, 2);
        g.C[c] = s.mloc();
        bytes += 16 * (R(c, 2) * s.mloc() + R(c, 2));
      }
      Scope sc(h, "adj_g4_gemv", bytes, 8 * (bytes / 16), st);
      launch_gemv_t(g, h->partials.p, (int64_t)h->partials.n, max_splits, st);
    } else {
      Scope sc(h, "adj_g4_zgemm", 0, 0, st);
      for (int c = 0; c < 3; ++c) {
        Zgemm z{};
        z.nbatch = 1;
        z.ta = kT;
        z.M[0] = s.mloc(); z.N[0] = k; z.K[0] = R(c, 2);
        z.A[0] = s.G4[c].p; z.lda[0] = R(c, 2);
        z.B[0] = s.z3.p + c * r3stride; z.ldb[0] = R(c, 2);
        z.C[0] = zout; z.ldc[0] = ldz;
        z.beta = c == 0 ? cmk(0, 0) : cmk(1, 0);
        launch_zgemm(z, nullptr, 0, st);
      }
      if (cj) {
        for (int j = 0; j < k; ++j) launch_conj(zout + ldz * j, s.mloc(), st);
      }
    }
  }
  if (h->comm) {
    // allgather of the column segments -> replicated z
    Scope sc(h, "nccl_allgather", 0, 0, st);
    cplx* seg = h->gather_buf.p + (int64_t)h->world * mp * k;
    const Shard& s = h->shards[0];
    if (s.mloc() < mp) {
      // zero the padding rows of the segment
      for (int j = 0; j < k; ++j)
        VSIE_CHECK_CUDA(cudaMemsetAsync(seg + mp * j + s.mloc(), 0, (mp - s.mloc()) * sizeof(cplx), st));
    }
    h->comm->allgather(reinterpret_cast<const double*>(seg), reinterpret_cast<double*>(h->gather_buf.p),
                       2 * (size_t)mp * k, st);
    // recv: [P][mp x k]; scatter into y (m x k, ld m)
    for (int p = 0; p < h->world; ++p) {
      const int64_t cb = std::min(m, mp * p), ce = std::min(m, mp * (p + 1));
      copy2d(y + cb, m, h->gather_buf.p + (int64_t)p * mp * k, mp, ce - cb, k, cudaMemcpyDeviceToDevice, st);
    }
  }
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
}
