// PWL (q = 12) coupling over four moment handles ("piecewise linear ... q = 12";
// P:381 the linear terms of Z_bc^f; reading R-PWL).
//
// Handle l (test_moment = l) holds the three chi blocks tested with the l-th PWL function of
// every voxel (1, (x - c_x)/h_x, (y - c_y)/h_y, (z - c_z)/h_z), each a TT of its own ranks
// (the q components are independent 4-D tensors).  Forward: the four applies write
// their blocks of y in place.  Transpose: the four m-vectors are summed on device in fixed
// order, z = ((z_0 + z_1) + z_2) + z_3.
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

}  // namespace

void apply_pwl(vsie_coupling_s* const hs[4], const cplx* x, cplx* y, int op, int nrhs, cudaStream_t st) {
  VSIE_REQUIRE(op == VSIE_OP_N || op == VSIE_OP_T || op == VSIE_OP_C, VSIE_ERR_ARG, "bad op");
  VSIE_REQUIRE(x != nullptr && y != nullptr, VSIE_ERR_ARG, "x / y is NULL");
  for (int l = 0; l < 4; ++l) {
    VSIE_REQUIRE(hs[l] != nullptr, VSIE_ERR_ARG, "apply_pwl: handle is NULL");
    VSIE_REQUIRE(hs[l]->test_moment == l, VSIE_ERR_ARG, "apply_pwl: h[l] must have test_moment l");
    const vsie_coupling_s* a = hs[0];
    const vsie_coupling_s* b = hs[l];
    bool same = a->m == b->m && a->world == b->world && a->rank == b->rank && a->loopback == b->loopback &&
                a->k0 == b->k0 && a->shards.size() == b->shards.size();
    for (int d = 0; d < 3 && same; ++d)
      same = a->grid.n[d] == b->grid.n[d] && a->grid.h[d] == b->grid.h[d] && a->grid.origin[d] == b->grid.origin[d];
    for (size_t q = 0; q < a->shards.size() && same; ++q)
      same = a->shards[q].i3b == b->shards[q].i3b && a->shards[q].i3e == b->shards[q].i3e;
    VSIE_REQUIRE(same, VSIE_ERR_ARG, "apply_pwl: handles differ in grid, sources or partition");
    VSIE_REQUIRE(nrhs >= 1 && nrhs <= b->nrhs_max, VSIE_ERR_ARG, "nrhs out of range");
  }
  const int64_t vox = local_vox(hs[0]) * nrhs, mm = hs[0]->m * nrhs;
  if (op == VSIE_OP_N) {
    for (int l = 0; l < 4; ++l) apply(hs[l], x, y + l * vox, op, nrhs, st);
    return;
  }
  hs[0]->pwl_scratch.ensure(3 * mm);
  cplx* s = hs[0]->pwl_scratch.p;
  apply(hs[0], x, y, op, nrhs, st);
  for (int l = 1; l < 4; ++l) apply(hs[l], x + l * vox, s + (l - 1) * mm, op, nrhs, st);
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(mm, 256)), 148 * 8);
  k_sum_moments<<<blocks, 256, 0, st>>>(y, s, mm);
  VSIE_CHECK_LAUNCH();
  ++hs[0]->apply_launches;
}

}  // namespace vsie
