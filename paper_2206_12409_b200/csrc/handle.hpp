// The coupling handle: geometry on device, TT cores laid out for the slab
// partition (SURVEY §8e design iii), apply workspaces, communicator, timers.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "comm.hpp"
#include "geometry.hpp"
#include "kernels.cuh"

namespace vsie {

// One rank's slab: voxel planes i3 in [i3b, i3e) and G4 columns [cb, ce).
struct Shard {
  int i3b = 0, i3e = 0;
  int64_t cb = 0, ce = 0;
  DevBuf<cplx> G3[3];   // (r2, i3e - i3b, r3) column-major: the owned i3 slice of G3
  DevBuf<cplx> G4[3];   // (r3, ce - cb): the owned columns of G4
  // G3 slice re-blocked for k_seg_gemv: g3b_ns row blocks [R q / ns, R (q + 1) / ns) of the
  // (r2 n3loc) x r3 matrix, block q stored column-major (L_q x r3) at offset r3 * row0_q,
  // so that every CTA streams one contiguous range
  DevBuf<cplx> G3b[3];
  int g3b_ns = 0;
  // apply workspaces (sized for nrhs_max)
  DevBuf<cplx> y4;      // [3][r3max * nrhs]  forward: G4 x partial / reduced
  DevBuf<cplx> Y3;      // [3][r2 * n3loc * nrhs]
  DevBuf<cplx> Y2;      // [3][r1 * n2 * n3loc * nrhs]
  DevBuf<cplx> W1;      // [3][r1 * n2 * n3loc * nrhs]   (adjoint: G1^T u)
  DevBuf<cplx> W2;      // [3][r2 * n3loc * nrhs]
  DevBuf<cplx> z3;      // [3][r3max * nrhs]
  DevBuf<cplx> zpart;   // [3][mloc_max * nrhs]  transpose: per-chi G4_chi^T z3_chi
  int n3loc() const { return i3e - i3b; }
  int64_t mloc() const { return ce - cb; }
};

struct Timed {
  std::string name;
  cudaEvent_t e0, e1;
  int64_t bytes, flops;
  int chi = -1;
  int call = 0;
  cudaEvent_t origin = nullptr;  // start of the apply call (trace mode)
};

// A captured apply (CUDA graph) for one (op, nrhs, x, y) combination.
struct GraphEntry {
  int op = 0, nrhs = 0;
  const void* x = nullptr;
  void* y = nullptr;
  const void* u = nullptr;   // second input / output of the fused pair
  void* z = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  uint64_t last_use = 0;
};

}  // namespace vsie

struct vsie_coupling_s {
  vsie::GridDesc grid{};
  int64_t m = 0;
  double k0 = 0;
  double scale_re = 1, scale_im = 0;
  vsie::Sources sources;
  uint64_t src_hash = 0;   // FNV-1a of the source table (PWL moment handles must agree)
  vsie::DevBuf<double> d_src;
  vsie::EntryGeom eg{};
  int ranks[3][3] = {{0}};
  bool has_cores = false;
  vsie::DevBuf<vsie::cplx> G1[3], G2[3];  // replicated on every rank
  std::vector<vsie::Shard> shards;         // 1 shard (own rank) or `world` (loopback)
  int rank = 0, world = 1, loopback = 0, device = 0;
  int nrhs_max = 64;
  int quad_rule = 0;                       // vsie_build_opts.quad_rule
  int test_moment = 0;                     // PWL test moment (vsie_build_opts.test_moment)
  std::unique_ptr<vsie::Comm> comm;
  vsie::DevBuf<vsie::cplx> partials;       // [3][partials_per_chi]
  int64_t partials_per_chi = 0;
  vsie::DevBuf<vsie::cplx> zgemm_ws;       // [3][zgemm_ws_per_chi]
  int64_t zgemm_ws_per_chi = 0;
  // apply orchestration: one stream per chi chain, fork/join events, graph cache
  cudaStream_t chi_stream[3] = {nullptr, nullptr, nullptr};
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  std::vector<vsie::GraphEntry> graphs;
  uint64_t graph_clock = 0;
  int use_graphs = 1;
  int pair_sched = 0;   // GMRES pair: 0 auto (fewer bytes), 1 G4 read once, 2 G3 read once
  vsie::DevBuf<vsie::cplx> gather_buf;     // allgather staging of z
  vsie::DevBuf<vsie::cplx> io_x, io_y;     // apply_host staging
  vsie::DevBuf<vsie::cplx> pwl_scratch;    // vsie_coupling_apply_pwl: Z_l^T u_l, l = 1..3
  vsie::DevBuf<int64_t> io_idx;
  cudaStream_t io_stream = nullptr;
  cudaStream_t pwl_stream = nullptr;   // apply_pair_pwl: this moment handle's pair runs here
  cudaEvent_t pwl_ev_fork = nullptr, pwl_ev_done = nullptr;
  cudaStream_t io_stream2 = nullptr;   // host pair: the transpose's copies + apply
  // info
  int64_t entries_evaluated = 0;
  int sweeps[3] = {0, 0, 0};
  double heldout_err[3] = {0, 0, 0};
  double build_s = 0, build_entry_s = 0, build_factor_s = 0, build_maxvol_s = 0;
  int64_t apply_launches = 0, apply_calls = 0;
  // timing
  int timing = 0;                 // 0 off, 1 serialised per-kernel timing, 2 concurrent timeline
  int scope_chi = -1;             // chain of the kernels being launched (trace records)
  int trace_call = 0;
  cudaEvent_t trace_origin = nullptr;
  std::vector<cudaEvent_t> origins;
  std::vector<vsie::Timed> pending;
  std::vector<vsie::TimerSlot> timers;
  std::vector<cudaEvent_t> event_pool;

  ~vsie_coupling_s();
};

namespace vsie {

// setup helpers (capi.cpp / cross.cpp)
void handle_init_geometry(vsie_coupling_s* h, const vsie_grid* grid, const vsie_mesh* meshes, int n_meshes,
                          double freq, const vsie_build_opts* opts);
void handle_partition(vsie_coupling_s* h);
void slab_partition(int n3, int64_t m, int world, int rank, int slab[2], int64_t cols[2]);
// installs full cores (host, column-major) for component chi; keeps the owned shards
void handle_set_cores_host(vsie_coupling_s* h, int chi, const int r[3], const cplx* const host[4]);
// same from device buffers (full cores on this device)
void handle_set_cores_device(vsie_coupling_s* h, int chi, const int r[3], const cplx* const dev[4]);
void handle_alloc_workspace(vsie_coupling_s* h);

void apply(vsie_coupling_s* h, const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st);
// y = Z x and z = Z^T u (adj_op OP_T) or Z^H u (OP_C) in one call, single RHS
void apply_pair(vsie_coupling_s* h, const cplx* x, cplx* y, const cplx* u, cplx* z, int adj_op, cudaStream_t st);
// vsie_coupling_apply_pwl (pwl.cu)
void apply_pwl(vsie_coupling_s* const hs[4], const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st);
void apply_pair_pwl(vsie_coupling_s* const hs[4], const cplx* x, cplx* y, const cplx* u, cplx* z, int adj_op,
                    cudaStream_t st);
// schedule the pair runs with: 1 = G4-shared, 2 = G3-shared (apply.cu)
int pair_schedule(vsie_coupling_s* h);
// drops the cached apply graphs (cores / workspaces changed)
void apply_reset_graphs(vsie_coupling_s* h);
void apply_destroy(vsie_coupling_s* h);
void tt_eval(vsie_coupling_s* h, const int64_t* idx, int64_t count, cplx* out, cudaStream_t st);
void launch_tt_eval(const cplx* const G[4], const int r[3], const int n[3], int64_t m, int chi_sel,
                    const int64_t* idx, int64_t count, int64_t nv, cplx* out, cudaStream_t st);

}  // namespace vsie
