// C ABI of the Z_bc coupling library (include/vsie_coupling.h).  Every entry
// point converts exceptions into status codes and records a thread-local
// message; no C++ exception crosses the boundary.
#include <algorithm>
#include <chrono>
#include <memory>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include "cross.hpp"
#include "farfar.hpp"
#include "farnear.hpp"
#include "handle.hpp"
#include "hybrid.hpp"

using namespace vsie;

namespace vsie {

AllocHook& alloc_hook() {
  static AllocHook h;
  return h;
}

void* dev_alloc_bytes(size_t bytes, AllocHook& used) {
  used = alloc_hook();
  void* p = nullptr;
  if (!used.alloc) {
    VSIE_CHECK_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  p = used.alloc(bytes, used.ctx);
  VSIE_REQUIRE(p != nullptr, VSIE_ERR_NOMEM,
               "device allocation hook returned NULL for " + std::to_string(bytes) + " bytes");
  VSIE_REQUIRE(reinterpret_cast<uintptr_t>(p) % 256 == 0, VSIE_ERR_ARG, "device allocation hook: pointer not 256-B aligned");
  return p;
}

void dev_free_bytes(void* p, const AllocHook& used) {
  if (!used.free) {
    cudaFree(p);
    return;
  }
  // cudaFree's ordering: work already queued on any stream may still use p, and a caching
  // allocator hands p out again at once
  cudaDeviceSynchronize();
  used.free(p, used.ctx);
}

}  // namespace vsie

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(VSIE_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(VSIE_ERR_CUDA, e.what());
  }
}

vsie_build_opts resolve_opts(const vsie_build_opts* o) {
  vsie_build_opts d;
  vsie_build_opts_default(&d);
  if (o) d = *o;
  VSIE_REQUIRE(d.max_rank >= 1 && d.max_sweeps >= 1 && d.oversample >= 1 && d.heldout >= 0, VSIE_ERR_ARG,
               "bad build options");
  VSIE_REQUIRE(std::isfinite(d.scale_re) && std::isfinite(d.scale_im), VSIE_ERR_ARG, "bad scale");
  return d;
}

void finish_handle(vsie_coupling_s* h) {
  handle_alloc_workspace(h);
  h->has_cores = true;
  VSIE_CHECK_CUDA(cudaDeviceSynchronize());
}

}  // namespace

extern "C" {

int32_t vsie_abi_version(void) { return VSIE_ABI_VERSION; }

int32_t vsie_set_allocator(void* (*dev_alloc)(size_t, void*), void (*dev_free)(void*, void*), void* ctx) {
  return guarded([&] {
    VSIE_REQUIRE((dev_alloc == nullptr) == (dev_free == nullptr), VSIE_ERR_ARG,
                 "dev_alloc and dev_free must both be set or both be NULL");
    AllocHook& h = alloc_hook();
    h.alloc = dev_alloc;
    h.free = dev_free;
    h.ctx = dev_alloc ? ctx : nullptr;
    return VSIE_OK;
  });
}

void vsie_build_opts_default(vsie_build_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->max_rank = 2048;
  o->max_sweeps = 8;
  o->oversample = 16;
  o->direct_svd_max = 384;
  o->heldout = 1000;
  o->nrhs_max = 64;
  o->seed = 12409010ull;
  o->scale_re = 1.0;
  o->scale_im = 0.0;
  o->rank = 0;
  o->world = 1;
  o->loopback = 0;
  o->nccl_unique_id = nullptr;
  o->device = -1;
  o->verbose = 0;
  o->test_moment = 0;
  o->quad_rule = 0;
}

const char* vsie_status_string(int32_t s) {
  switch (s) {
    case VSIE_OK: return "VSIE_OK";
    case VSIE_WARN_NOT_CONVERGED: return "VSIE_WARN_NOT_CONVERGED";
    case VSIE_ERR_ARG: return "VSIE_ERR_ARG";
    case VSIE_ERR_GEOMETRY: return "VSIE_ERR_GEOMETRY";
    case VSIE_ERR_CUDA: return "VSIE_ERR_CUDA";
    case VSIE_ERR_NOMEM: return "VSIE_ERR_NOMEM";
    case VSIE_ERR_NCCL: return "VSIE_ERR_NCCL";
    case VSIE_ERR_STATE: return "VSIE_ERR_STATE";
    default: return "VSIE_UNKNOWN_STATUS";
  }
}

const char* vsie_last_error_message(void) { return g_last_error.c_str(); }

int32_t vsie_slab_partition(int32_t n3, int64_t m, int32_t world, int32_t rank, int32_t slab[2], int64_t cols[2]) {
  return guarded([&] {
    VSIE_REQUIRE(slab != nullptr && cols != nullptr, VSIE_ERR_ARG, "NULL argument");
    VSIE_REQUIRE(world >= 1 && rank >= 0 && rank < world && n3 >= world && m >= 1, VSIE_ERR_ARG,
                 "bad partition arguments");
    slab_partition(n3, m, world, rank, slab, cols);
    return VSIE_OK;
  });
}

int32_t vsie_nccl_unique_id(void* out128) {
  return guarded([&] {
    VSIE_REQUIRE(out128 != nullptr, VSIE_ERR_ARG, "out is NULL");
    return nccl_unique_id(out128);
  });
}

int32_t vsie_coupling_build(const vsie_grid* grid, const vsie_mesh* meshes, int32_t n_meshes, double freq_hz,
                            double tol, const vsie_build_opts* opts, vsie_coupling_t* out) {
  if (out) *out = nullptr;
  return guarded([&] {
    VSIE_REQUIRE(out != nullptr, VSIE_ERR_ARG, "out is NULL");
    VSIE_REQUIRE(tol > 0 && tol < 1 && std::isfinite(tol), VSIE_ERR_ARG, "tol must be in (0, 1)");
    const vsie_build_opts o = resolve_opts(opts);
    auto t0 = std::chrono::steady_clock::now();
    auto h = std::make_unique<vsie_coupling_s>();
    handle_init_geometry(h.get(), grid, meshes, n_meshes, freq_hz, &o);
    const int status = cross_build(h.get(), tol, o);
    finish_handle(h.get());
    h->build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
    return status;
  });
}

int32_t vsie_coupling_import_cores(const vsie_grid* grid, const vsie_mesh* meshes, int32_t n_meshes,
                                   double freq_hz, const int32_t ranks[9], const void* const host_cores[12],
                                   const vsie_build_opts* opts, vsie_coupling_t* out) {
  if (out) *out = nullptr;
  return guarded([&] {
    VSIE_REQUIRE(out != nullptr && ranks != nullptr && host_cores != nullptr, VSIE_ERR_ARG, "NULL argument");
    const vsie_build_opts o = resolve_opts(opts);
    auto h = std::make_unique<vsie_coupling_s>();
    handle_init_geometry(h.get(), grid, meshes, n_meshes, freq_hz, &o);
    for (int c = 0; c < 3; ++c) {
      const int r[3] = {ranks[3 * c], ranks[3 * c + 1], ranks[3 * c + 2]};
      const cplx* src[4];
      for (int k = 0; k < 4; ++k) src[k] = static_cast<const cplx*>(host_cores[4 * c + k]);
      handle_set_cores_host(h.get(), c, r, src);
    }
    finish_handle(h.get());
    *out = h.release();
    return VSIE_OK;
  });
}

int32_t vsie_coupling_export_cores(vsie_coupling_t h, int32_t chi, int32_t k, void* host_dst, int64_t* nelems) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && nelems != nullptr, VSIE_ERR_ARG, "NULL argument");
    VSIE_REQUIRE(h->has_cores, VSIE_ERR_STATE, "handle has no TT cores");
    VSIE_REQUIRE(chi >= 0 && chi < 3 && k >= 0 && k < 4, VSIE_ERR_ARG, "chi / k out of range");
    VSIE_REQUIRE(h->comm == nullptr, VSIE_ERR_STATE, "export_cores of a multi-process handle: export per rank");
    const int n[4] = {h->grid.n[0], h->grid.n[1], h->grid.n[2], (int)h->m};
    const int64_t rl = k == 0 ? 1 : h->ranks[chi][k - 1];
    const int64_t rr = k == 3 ? 1 : h->ranks[chi][k];
    const int64_t total = rl * n[k] * rr;
    *nelems = total;
    if (!host_dst) return VSIE_OK;
    cplx* dst = static_cast<cplx*>(host_dst);
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    if (k == 0) {
      VSIE_CHECK_CUDA(cudaMemcpy(dst, h->G1[chi].p, total * sizeof(cplx), cudaMemcpyDeviceToHost));
    } else if (k == 1) {
      VSIE_CHECK_CUDA(cudaMemcpy(dst, h->G2[chi].p, total * sizeof(cplx), cudaMemcpyDeviceToHost));
    } else if (k == 2) {
      const int64_t r2 = rl, r3 = rr, n3 = n[2];
      for (const Shard& s : h->shards) {
        const int64_t n3l = s.n3loc();
        if (n3l == 0) continue;
        VSIE_CHECK_CUDA(cudaMemcpy2D(dst + r2 * s.i3b, r2 * n3 * sizeof(cplx), s.G3[chi].p, r2 * n3l * sizeof(cplx),
                                     r2 * n3l * sizeof(cplx), r3, cudaMemcpyDeviceToHost));
      }
    } else {
      const int64_t r3 = rl;
      for (const Shard& s : h->shards)
        if (s.mloc() > 0)
          VSIE_CHECK_CUDA(cudaMemcpy(dst + r3 * s.cb, s.G4[chi].p, r3 * s.mloc() * sizeof(cplx),
                                     cudaMemcpyDeviceToHost));
    }
    return VSIE_OK;
  });
}

int32_t vsie_coupling_round(vsie_coupling_t h, double tol) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    return tt_round(h, tol);
  });
}

int32_t vsie_coupling_apply(vsie_coupling_t h, const void* x, void* y, int32_t op, int32_t nrhs, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    apply(h, static_cast<const cplx*>(x), static_cast<cplx*>(y), op, nrhs, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_apply_host(vsie_coupling_t h, const void* x_host, void* y_host, int32_t op, int32_t nrhs) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && x_host != nullptr && y_host != nullptr, VSIE_ERR_ARG, "NULL argument");
    VSIE_REQUIRE(nrhs >= 1 && nrhs <= h->nrhs_max, VSIE_ERR_ARG, "nrhs out of range");
    const int64_t n12 = (int64_t)h->grid.n[0] * h->grid.n[1];
    int64_t vox = 0;
    if (h->comm)
      vox = 3 * n12 * h->shards[0].n3loc();
    else
      vox = 3 * h->grid.nv();
    const int64_t nx = (op == VSIE_OP_N ? h->m : vox) * nrhs;
    const int64_t ny = (op == VSIE_OP_N ? vox : h->m) * nrhs;
    h->io_x.ensure(nx);
    h->io_y.ensure(ny);
    if (!h->io_stream) VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->io_stream, cudaStreamNonBlocking));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(h->io_x.p, x_host, nx * sizeof(cplx), cudaMemcpyHostToDevice, h->io_stream));
    apply(h, h->io_x.p, h->io_y.p, op, nrhs, h->io_stream);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(y_host, h->io_y.p, ny * sizeof(cplx), cudaMemcpyDeviceToHost, h->io_stream));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(h->io_stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_apply_pwl(const vsie_coupling_t h[4], const void* x, void* y, int32_t op, int32_t nrhs,
                                void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle array is NULL");
    vsie_coupling_s* hs[4] = {h[0], h[1], h[2], h[3]};
    apply_pwl(hs, static_cast<const cplx*>(x), static_cast<cplx*>(y), op, nrhs, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_apply_pair_pwl(const vsie_coupling_t h[4], const void* x, void* y, const void* u, void* z,
                                     int32_t adj_op, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle array is NULL");
    vsie_coupling_s* hs[4] = {h[0], h[1], h[2], h[3]};
    apply_pair_pwl(hs, static_cast<const cplx*>(x), static_cast<cplx*>(y), static_cast<const cplx*>(u),
                   static_cast<cplx*>(z), adj_op, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_apply_pair(vsie_coupling_t h, const void* x, void* y, const void* u, void* z, int32_t adj_op,
                                 void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    apply_pair(h, static_cast<const cplx*>(x), static_cast<cplx*>(y), static_cast<const cplx*>(u), static_cast<cplx*>(z),
               adj_op, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_apply_pair_host(vsie_coupling_t h, const void* x_host, void* y_host, const void* u_host,
                                      void* z_host, int32_t adj_op) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && x_host && y_host && u_host && z_host, VSIE_ERR_ARG, "NULL argument");
    const int64_t n12 = (int64_t)h->grid.n[0] * h->grid.n[1];
    const int64_t vox = h->comm ? 3 * n12 * h->shards[0].n3loc() : 3 * h->grid.nv();
    h->io_x.ensure(h->m + vox);
    h->io_y.ensure(vox + h->m);
    if (!h->io_stream) VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->io_stream, cudaStreamNonBlocking));
    cplx* dx = h->io_x.p;
    cplx* du = h->io_x.p + h->m;
    cplx* dy = h->io_y.p;
    cplx* dz = h->io_y.p + vox;
    if (!h->comm) {
      // Host buffers: the PCIe copies dominate (2 x 16 * 3 n_v bytes against ~0.1 ms of
      // device work), and y = Z x needs only x.  So the forward runs first on one stream
      // and its voxel result streams back (D2H) while u streams in (H2D) on a second
      // stream for the transpose: the two large copies overlap in opposite directions.
      // The two applies use disjoint workspaces (the transpose's Ctx::ws offset).
      if (!h->io_stream2) VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->io_stream2, cudaStreamNonBlocking));
      VSIE_CHECK_CUDA(cudaMemcpyAsync(dx, x_host, h->m * sizeof(cplx), cudaMemcpyHostToDevice, h->io_stream));
      apply(h, dx, dy, VSIE_OP_N, 1, h->io_stream);
      VSIE_CHECK_CUDA(cudaMemcpyAsync(y_host, dy, vox * sizeof(cplx), cudaMemcpyDeviceToHost, h->io_stream));
      VSIE_CHECK_CUDA(cudaMemcpyAsync(du, u_host, vox * sizeof(cplx), cudaMemcpyHostToDevice, h->io_stream2));
      apply(h, du, dz, adj_op, 1, h->io_stream2);
      VSIE_CHECK_CUDA(cudaMemcpyAsync(z_host, dz, h->m * sizeof(cplx), cudaMemcpyDeviceToHost, h->io_stream2));
      VSIE_CHECK_CUDA(cudaStreamSynchronize(h->io_stream));
      VSIE_CHECK_CUDA(cudaStreamSynchronize(h->io_stream2));
      return VSIE_OK;
    }
    VSIE_CHECK_CUDA(cudaMemcpyAsync(dx, x_host, h->m * sizeof(cplx), cudaMemcpyHostToDevice, h->io_stream));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(du, u_host, vox * sizeof(cplx), cudaMemcpyHostToDevice, h->io_stream));
    apply_pair(h, dx, dy, du, dz, adj_op, h->io_stream);
    VSIE_CHECK_CUDA(cudaMemcpyAsync(y_host, dy, vox * sizeof(cplx), cudaMemcpyDeviceToHost, h->io_stream));
    VSIE_CHECK_CUDA(cudaMemcpyAsync(z_host, dz, h->m * sizeof(cplx), cudaMemcpyDeviceToHost, h->io_stream));
    VSIE_CHECK_CUDA(cudaStreamSynchronize(h->io_stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_entries(vsie_coupling_t h, const int64_t* idx, int64_t count, void* out, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    VSIE_REQUIRE(count >= 0, VSIE_ERR_ARG, "count < 0");
    if (count == 0) return VSIE_OK;
    VSIE_REQUIRE(idx != nullptr && out != nullptr, VSIE_ERR_ARG, "idx / out is NULL");
    launch_entries_list(h->eg, idx, count, static_cast<cplx*>(out), static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_supercore(vsie_coupling_t h, int32_t chi, int32_t k, const int32_t* left, int32_t n_left,
                                const int32_t* right, int32_t n_right, void* out, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && out != nullptr, VSIE_ERR_ARG, "handle / out is NULL");
    VSIE_REQUIRE(chi >= 0 && chi < 3 && k >= 1 && k <= 3, VSIE_ERR_ARG, "chi / k out of range");
    VSIE_REQUIRE(n_left >= 1 && n_right >= 1, VSIE_ERR_ARG, "n_left / n_right < 1");
    VSIE_REQUIRE(k == 1 || left != nullptr, VSIE_ERR_ARG, "left is NULL");
    VSIE_REQUIRE(k == 3 || right != nullptr, VSIE_ERR_ARG, "right is NULL");
    VSIE_REQUIRE(k != 1 || n_left == 1, VSIE_ERR_ARG, "k = 1 has n_left = 1");
    VSIE_REQUIRE(k != 3 || n_right == 1, VSIE_ERR_ARG, "k = 3 has n_right = 1");
    const int64_t dims[4] = {h->grid.n[0], h->grid.n[1], h->grid.n[2], h->m};
    BlockDesc b{};
    b.chi = chi;
    b.k = k;
    b.rl = n_left;
    b.nk = dims[k - 1];
    b.nk1 = dims[k];
    b.rr = n_right;
    b.left = left;
    b.right = right;
    b.col0 = 0;
    b.col1 = b.nk1 * b.rr;
    b.ld = b.rl * b.nk;
    launch_entries_block(h->eg, b, static_cast<cplx*>(out), static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_tt_eval(vsie_coupling_t h, const int64_t* idx, int64_t count, void* out, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    VSIE_REQUIRE(count >= 0, VSIE_ERR_ARG, "count < 0");
    if (count == 0) return VSIE_OK;
    VSIE_REQUIRE(idx != nullptr && out != nullptr, VSIE_ERR_ARG, "idx / out is NULL");
    tt_eval(h, idx, count, static_cast<cplx*>(out), static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_coupling_info(vsie_coupling_t h, vsie_info* out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && out != nullptr, VSIE_ERR_ARG, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    for (int a = 0; a < 3; ++a) out->n[a] = h->grid.n[a];
    out->m = h->m;
    int64_t core_elems = 0, bytes = 0;
    for (int c = 0; c < 3; ++c) {
      for (int k = 0; k < 3; ++k) out->ranks[c][k] = h->ranks[c][k];
      const int64_t r1 = h->ranks[c][0], r2 = h->ranks[c][1], r3 = h->ranks[c][2];
      core_elems += h->grid.n[0] * r1 + r1 * h->grid.n[1] * r2 + r2 * h->grid.n[2] * r3 + r3 * h->m;
      bytes += h->G1[c].bytes() + h->G2[c].bytes();
      for (const Shard& s : h->shards) bytes += s.G3[c].bytes() + s.G4[c].bytes();
      out->sweeps[c] = h->sweeps[c];
      out->heldout_err[c] = h->heldout_err[c];
    }
    out->core_bytes = bytes;
    if (h->has_cores && core_elems > 0) {
      int64_t num = 3 * h->grid.nv() * h->m, den = core_elems;
      const int64_t g = std::gcd(num, den);
      out->compression_num = num / g;
      out->compression_den = den / g;
    }
    out->entries_evaluated = h->entries_evaluated;
    out->build_s = h->build_s;
    out->build_entry_s = h->build_entry_s;
    out->build_factor_s = h->build_factor_s;
    out->build_maxvol_s = h->build_maxvol_s;
    out->slab[0] = h->shards.empty() ? 0 : h->shards.front().i3b;
    out->slab[1] = h->shards.empty() ? 0 : h->shards.back().i3e;
    out->cols[0] = h->shards.empty() ? 0 : h->shards.front().cb;
    out->cols[1] = h->shards.empty() ? 0 : h->shards.back().ce;
    out->world = h->world;
    out->rank = h->rank;
    out->loopback = h->loopback;
    out->k0 = h->k0;
    out->apply_launches = h->apply_launches;
    out->apply_calls = h->apply_calls;
    out->test_moment = h->test_moment;
    out->pair_schedule = h->has_cores ? pair_schedule(h) : 0;
    out->quad_rule = h->quad_rule;
    return VSIE_OK;
  });
}

int32_t vsie_coupling_set_timing(vsie_coupling_t h, int32_t enable) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    for (auto& t : h->pending) {
      h->event_pool.push_back(t.e0);
      h->event_pool.push_back(t.e1);
    }
    h->pending.clear();
    h->timers.clear();
    for (cudaEvent_t e : h->origins) cudaEventDestroy(e);
    h->origins.clear();
    h->trace_origin = nullptr;
    h->trace_call = 0;
    VSIE_REQUIRE(enable >= 0 && enable <= 2, VSIE_ERR_ARG, "timing mode must be 0, 1 or 2");
    h->timing = enable;
    // events are recorded inside stream captures, where they cannot be created
    while (enable && h->event_pool.size() < 4096) {
      cudaEvent_t e;
      VSIE_CHECK_CUDA(cudaEventCreate(&e));
      h->event_pool.push_back(e);
    }
    return VSIE_OK;
  });
}

int32_t vsie_coupling_timers(vsie_coupling_t h, vsie_timer* out, int32_t max, int32_t* n_out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && n_out != nullptr, VSIE_ERR_ARG, "NULL argument");
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    for (auto& t : h->pending) {
      float ms = 0;
      VSIE_CHECK_CUDA(cudaEventElapsedTime(&ms, t.e0, t.e1));
      TimerSlot* slot = nullptr;
      for (auto& s : h->timers)
        if (s.name == t.name) slot = &s;
      if (!slot) {
        h->timers.push_back(TimerSlot{t.name, 0, 0.0, t.bytes, t.flops});
        slot = &h->timers.back();
      }
      slot->launches += 1;
      slot->total_ms += ms;
      h->event_pool.push_back(t.e0);
      h->event_pool.push_back(t.e1);
    }
    h->pending.clear();
    const int n = (int)h->timers.size();
    *n_out = n;
    for (int i = 0; i < n && i < max && out; ++i) {
      std::memset(&out[i], 0, sizeof(vsie_timer));
      std::strncpy(out[i].name, h->timers[i].name.c_str(), sizeof(out[i].name) - 1);
      out[i].launches = h->timers[i].launches;
      out[i].total_ms = h->timers[i].total_ms;
      out[i].bytes_per_launch = h->timers[i].bytes;
      out[i].flops_per_launch = h->timers[i].flops;
    }
    return VSIE_OK;
  });
}

int32_t vsie_coupling_configure(vsie_coupling_t h, int32_t use_graphs, int32_t pair_schedule) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "handle is NULL");
    VSIE_REQUIRE(pair_schedule <= 2, VSIE_ERR_ARG, "pair_schedule must be 0 (auto), 1 (G4 shared) or 2 (G3 shared)");
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    if (use_graphs >= 0) h->use_graphs = use_graphs != 0;
    if (pair_schedule >= 0) h->pair_sched = pair_schedule;
    apply_reset_graphs(h);
    return VSIE_OK;
  });
}

int32_t vsie_coupling_trace(vsie_coupling_t h, vsie_trace* out, int32_t max, int32_t* n_out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && n_out != nullptr, VSIE_ERR_ARG, "NULL argument");
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    int n = 0;
    for (auto& t : h->pending) {
      if (t.origin && out && n < max) {
        float a = 0, b = 0;
        VSIE_CHECK_CUDA(cudaEventElapsedTime(&a, t.origin, t.e0));
        VSIE_CHECK_CUDA(cudaEventElapsedTime(&b, t.origin, t.e1));
        std::memset(&out[n], 0, sizeof(vsie_trace));
        std::strncpy(out[n].name, t.name.c_str(), sizeof(out[n].name) - 1);
        out[n].chi = t.chi;
        out[n].call = t.call;
        out[n].t0_ms = a;
        out[n].t1_ms = b;
        ++n;
      }
      h->event_pool.push_back(t.e0);
      h->event_pool.push_back(t.e1);
    }
    h->pending.clear();
    *n_out = n;
    return VSIE_OK;
  });
}

void vsie_coupling_destroy(vsie_coupling_t h) {
  if (!h) return;
  cudaDeviceSynchronize();
  delete h;
}

// ----------------------------------------------------------------- far-near block (vsie_farnear.h)
void vsie_farnear_opts_default(vsie_farnear_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->max_rank = 2048;
  o->scale_re = 1.0;
  o->scale_im = 0.0;
  o->device = -1;
  o->verbose = 0;
}

int32_t vsie_farnear_build(const vsie_mesh* near_meshes, int32_t n_near, const vsie_mesh* far_meshes, int32_t n_far,
                           double freq_hz, double tol, const vsie_farnear_opts* opts, vsie_farnear_t* out) {
  if (out) *out = nullptr;
  return guarded([&] {
    VSIE_REQUIRE(out != nullptr && near_meshes != nullptr && far_meshes != nullptr && n_near >= 1 && n_far >= 1,
                 VSIE_ERR_ARG, "farnear_build: NULL argument or no meshes");
    vsie_farnear_opts o;
    vsie_farnear_opts_default(&o);
    if (opts) o = *opts;
    std::unique_ptr<vsie_farnear_s> h(new vsie_farnear_s());
    const int st = farnear_build(near_meshes, n_near, far_meshes, n_far, freq_hz, tol, o, h.get());
    *out = h.release();
    return st;
  });
}

int32_t vsie_farnear_entries(vsie_farnear_t h, const int64_t* idx, int64_t count, void* out, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farnear_entries(h, idx, count, out, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_farnear_apply(vsie_farnear_t h, const void* x, void* y, int32_t op, int32_t nrhs, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farnear_apply(h, x, y, op, nrhs, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_farnear_apply_pair(vsie_farnear_t h, const void* x_far, void* y_near, const void* x_near, void* y_far,
                                void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farnear_apply_pair(h, x_far, y_near, x_near, y_far, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_farnear_export(vsie_farnear_t h, void* U_host, void* W_host, int32_t* rows, int32_t* cols) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    VSIE_CHECK_CUDA(cudaDeviceSynchronize());
    if (U_host && h->rank > 0) VSIE_CHECK_CUDA(cudaMemcpy(U_host, h->U.p, h->U.bytes(), cudaMemcpyDeviceToHost));
    if (W_host && h->rank > 0) VSIE_CHECK_CUDA(cudaMemcpy(W_host, h->W.p, h->W.bytes(), cudaMemcpyDeviceToHost));
    if (rows) std::copy(h->piv_i.begin(), h->piv_i.end(), rows);
    if (cols) std::copy(h->piv_j.begin(), h->piv_j.end(), cols);
    return VSIE_OK;
  });
}

int32_t vsie_farnear_get_info(vsie_farnear_t h, vsie_farnear_info* out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && out != nullptr, VSIE_ERR_ARG, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->m_near = h->mn;
    out->m_far = h->mf;
    out->rank = h->rank;
    out->stop = h->stop;
    out->est_err = h->est_err;
    out->frob = h->frob;
    out->min_distance = h->min_dist;
    out->max_edge = h->max_edge;
    out->k0 = h->k0;
    out->build_s = h->build_s;
    out->entries_evaluated = h->entries;
    out->factor_bytes = (int64_t)16 * h->rank * (h->mn + h->mf);
    out->apply_calls = h->apply_calls;
    return VSIE_OK;
  });
}

void vsie_farnear_destroy(vsie_farnear_t h) {
  if (!h) return;
  cudaDeviceSynchronize();
  delete h;
}

// ----------------------------------------------------------------- far-far block (vsie_farfar.h)
int32_t vsie_farfar_build(const vsie_mesh* meshes, int32_t n_meshes, double freq_hz, double scale_re, double scale_im,
                          int32_t device, vsie_farfar_t* out) {
  if (out) *out = nullptr;
  return guarded([&] {
    VSIE_REQUIRE(out != nullptr, VSIE_ERR_ARG, "farfar_build: NULL out");
    std::unique_ptr<vsie_farfar_s> h(new vsie_farfar_s());
    farfar_build(meshes, n_meshes, freq_hz, scale_re, scale_im, device, h.get());
    *out = h.release();
    return VSIE_OK;
  });
}

int32_t vsie_farfar_entries(vsie_farfar_t h, const int64_t* idx, int64_t count, void* out, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farfar_entries(h, idx, count, out, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_farfar_apply(vsie_farfar_t h, const void* x, void* y, int32_t op, int32_t nrhs, int32_t accumulate,
                          void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farfar_apply(h, x, y, op, nrhs, accumulate != 0, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_farfar_export(vsie_farfar_t h, void* host_dense) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    farfar_export(h, host_dense);
    return VSIE_OK;
  });
}

int32_t vsie_farfar_get_info(vsie_farfar_t h, vsie_farfar_info* out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && out != nullptr, VSIE_ERR_ARG, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    out->m = h->m;
    out->tile = 128;
    out->tiles = h->tiles;
    out->matrix_bytes = (int64_t)h->Z.bytes();
    out->near_pairs = h->near_pairs;
    out->build_s = h->build_s;
    out->k0 = h->k0;
    out->apply_calls = h->apply_calls;
    return VSIE_OK;
  });
}

void vsie_farfar_destroy(vsie_farfar_t h) {
  if (!h) return;
  cudaDeviceSynchronize();
  delete h;
}

}  // extern "C"

// ------------------------------------------------------------------ hybrid system + GMRES (vsie_hybrid.h)
extern "C" {

int32_t vsie_hybrid_create(vsie_farfar_t ff, vsie_farnear_t fn, vsie_farfar_t nn, vsie_coupling_t cb_far,
                           vsie_coupling_t cb_near, const void* d_body, vsie_hybrid_t* out) {
  return guarded([&] {
    VSIE_REQUIRE(out != nullptr, VSIE_ERR_ARG, "out is NULL");
    *out = nullptr;
    std::unique_ptr<vsie_hybrid_s, void (*)(vsie_hybrid_s*)> h(hybrid_new(), hybrid_delete);
    hybrid_create(ff, fn, nn, cb_far, cb_near, d_body, h.get());
    *out = h.release();
    return VSIE_OK;
  });
}

int32_t vsie_hybrid_matvec(vsie_hybrid_t h, const void* x, void* y, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    hybrid_matvec(h, x, y, static_cast<cudaStream_t>(stream));
    return VSIE_OK;
  });
}

int32_t vsie_hybrid_gmres(vsie_hybrid_t h, const void* b, void* x, int32_t restart, int32_t max_iter, double tol,
                          double* history, vsie_gmres_info* info, void* stream) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr, VSIE_ERR_ARG, "NULL handle");
    return hybrid_gmres(h, b, x, restart, max_iter, tol, history, info, static_cast<cudaStream_t>(stream));
  });
}

int32_t vsie_hybrid_get_info(vsie_hybrid_t h, vsie_hybrid_info* out) {
  return guarded([&] {
    VSIE_REQUIRE(h != nullptr && out != nullptr, VSIE_ERR_ARG, "NULL argument");
    hybrid_info(h, out);
    return VSIE_OK;
  });
}

void vsie_hybrid_destroy(vsie_hybrid_t h) {
  if (h) hybrid_delete(h);
}

}  // extern "C"
