// PWL (q = 12) coupling over four moment handles ("piecewise linear ... q = 12";
// P:381 the linear terms of Z_bc^f; reading R-PWL).
//
// Handle l (test_moment = l) holds the three chi blocks tested with the l-th PWL function of
// every voxel (1, (x - c_x)/h_x, (y - c_y)/h_y, (z - c_z)/h_z), each a TT of its own ranks
// (the q components are independent 4-D tensors).  Forward: the four applies write
// their blocks of y in place.  Transpose: the four m-vectors are summed on device in fixed
// order, z = ((z_0 + z_1) + z_2) + z_3.
#include <cstdlib>

#include "handle.hpp"
#include "kernels.cuh"

namespace vsie {
namespace {

__global__ void __launch_bounds__(256) k_sum_moments(cplx* __restrict__ z, const cplx* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    cplx a = z[i];
    a = cadd(a, s[i]);
    a = cadd(a, s[i + n]);
    a = cadd(a, s[i + 2 * n]);
    z[i] = a;
  }
}

int64_t local_vox(const vsie_coupling_s* h) {
  const int64_t n12 = (int64_t)h->grid.n[0] * h->grid.n[1];
  return h->comm ? 3 * n12 * h->shards[0].n3loc() : 3 * h->grid.nv();
}

void check_pwl(vsie_coupling_s* const hs[4], int nrhs) {
  for (int l = 0; l < 4; ++l) {
    VSIE_REQUIRE(hs[l] != nullptr, VSIE_ERR_ARG, "apply_pwl: handle is NULL");
    VSIE_REQUIRE(hs[l]->test_moment == l, VSIE_ERR_ARG, "apply_pwl: h[l] must have test_moment l");
    const vsie_coupling_s* a = hs[0];
    const vsie_coupling_s* b = hs[l];
    bool same = a->m == b->m && a->world == b->world && a->rank == b->rank && a->loopback == b->loopback &&
                a->k0 == b->k0 && a->scale_re == b->scale_re && a->scale_im == b->scale_im &&
                a->src_hash == b->src_hash && a->shards.size() == b->shards.size();
    for (int d = 0; d < 3 && same; ++d)
      same = a->grid.n[d] == b->grid.n[d] && a->grid.h[d] == b->grid.h[d] && a->grid.origin[d] == b->grid.origin[d];
    for (size_t q = 0; q < a->shards.size() && same; ++q)
      same = a->shards[q].i3b == b->shards[q].i3b && a->shards[q].i3e == b->shards[q].i3e;
    VSIE_REQUIRE(same, VSIE_ERR_ARG, "apply_pwl: handles differ in grid, sources or partition");
    VSIE_REQUIRE(nrhs >= 1 && nrhs <= b->nrhs_max, VSIE_ERR_ARG, "nrhs out of range");
  }
}

void sum_moments(vsie_coupling_s* h0, cplx* z, const cplx* s, int64_t mm, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(mm, 256)), 148 * 8);
  k_sum_moments<<<blocks, 256, 0, st>>>(z, s, mm);
  VSIE_CHECK_LAUNCH();
  ++h0->apply_launches;
}

// One process: the four moment handles run on four streams, so one
// handle's latency-bound G1 / G2 phases overlap the others' HBM-bound G3 / G4 passes.
// Multi-process handles (own NCCL communicator each) run one after another: collectives
// of different communicators issued concurrently may wait on each other's SMs.
void pwl_fork(vsie_coupling_s* const hs[4], cudaStream_t st) {
  for (int l = 0; l < 4; ++l) {
    vsie_coupling_s* h = hs[l];
    if (!h->pwl_stream) {
      VSIE_CHECK_CUDA(cudaStreamCreateWithFlags(&h->pwl_stream, cudaStreamNonBlocking));
      VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->pwl_ev_fork, cudaEventDisableTiming));
      VSIE_CHECK_CUDA(cudaEventCreateWithFlags(&h->pwl_ev_done, cudaEventDisableTiming));
    }
  }
  VSIE_CHECK_CUDA(cudaEventRecord(hs[0]->pwl_ev_fork, st));
  for (int l = 0; l < 4; ++l) VSIE_CHECK_CUDA(cudaStreamWaitEvent(hs[l]->pwl_stream, hs[0]->pwl_ev_fork, 0));
}

void pwl_join(vsie_coupling_s* const hs[4], cudaStream_t st) {
  for (int l = 0; l < 4; ++l) {
    VSIE_CHECK_CUDA(cudaEventRecord(hs[l]->pwl_ev_done, hs[l]->pwl_stream));
    VSIE_CHECK_CUDA(cudaStreamWaitEvent(st, hs[l]->pwl_ev_done, 0));
  }
}

}  // namespace

void apply_pwl(vsie_coupling_s* const hs[4], const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st) {
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "bad op");
  VSIE_REQUIRE(x != nullptr && y != nullptr, VSIE_ERR_ARG, "x / y is NULL");
  check_pwl(hs, nrhs);
  const int64_t vox = local_vox(hs[0]) * nrhs, mm = hs[0]->m * nrhs;
  cplx* s = nullptr;
  if (op != VSIE_OP_N) {
    hs[0]->pwl_scratch.ensure(3 * mm);
    s = hs[0]->pwl_scratch.p;
  }
  const bool conc = !hs[0]->comm;
  if (conc) pwl_fork(hs, st);
  for (int l = 0; l < 4; ++l) {
    cudaStream_t sl = conc ? hs[l]->pwl_stream : st;
    if (op == VSIE_OP_N)
      apply(hs[l], x, y + l * vox, op, nrhs, sl);
    else
      apply(hs[l], x + l * vox, l == 0 ? y : s + (l - 1) * mm, op, nrhs, sl);
  }
  if (conc) pwl_join(hs, st);
  if (op != VSIE_OP_N) sum_moments(hs[0], y, s, mm, st);
}

// The q = 12 GMRES coupling pair: y = Z_pwl x and z = Z_pwl^op u, each moment handle's
// fused pair (one G4 pass per handle for both directions), then the fixed-order z sum.
void apply_pair_pwl(vsie_coupling_s* const hs[4], const cplx* x, cplx* y, const cplx* u, cplx* z, int adj_op,
                    cudaStream_t st) {
  VSIE_REQUIRE(adj_op == VSIE_OP_T || adj_op == VSIE_OP_C, VSIE_ERR_ARG, "adj_op must be OP_T or OP_C");
  VSIE_REQUIRE(x && y && u && z, VSIE_ERR_ARG, "x / y / u / z is NULL");
  check_pwl(hs, 1);
  const int64_t vox = local_vox(hs[0]), mm = hs[0]->m;
  hs[0]->pwl_scratch.ensure(3 * mm);
  cplx* s = hs[0]->pwl_scratch.p;
  if (hs[0]->comm) {
    apply_pair(hs[0], x, y, u, z, adj_op, st);
    for (int l = 1; l < 4; ++l) apply_pair(hs[l], x, y + l * vox, u + l * vox, s + (l - 1) * mm, adj_op, st);
  } else {
    pwl_fork(hs, st);
    for (int l = 0; l < 4; ++l)
      apply_pair(hs[l], x, y + l * vox, u + l * vox, l == 0 ? z : s + (l - 1) * mm, adj_op, hs[l]->pwl_stream);
    pwl_join(hs, st);
  }
  sum_moments(hs[0], z, s, mm, st);
}

}  // namespace vsie
