// Far-near conductor block (farnear.cu): the handle behind include/vsie_farnear.h.
#pragma once

#include <vector>

#include "../../include/vsie_farnear.h"
#include "kernels.cuh"

struct vsie_farnear_s {
  int device = 0;
  int64_t mn = 0, mf = 0;
  int rank = 0, stop = 0;
  double est_err = 0, frob = 0, min_dist = 0, max_edge = 0, k0 = 0, build_s = 0;
  double scale_re = 1, scale_im = 0;
  int64_t entries = 0, apply_calls = 0;
  vsie::DevBuf<double> src_n, src_f;   // [m][36] near (rows) / far (columns)
  vsie::DevBuf<vsie::cplx> U, W;       // column-major m_n x rank, m_f x rank
  std::vector<int> piv_i, piv_j;
  // apply workspaces
  vsie::DevBuf<vsie::cplx> part, t;
  vsie::DevBuf<unsigned> counters;
  vsie::DevBuf<vsie::cplx> gemm_ws, xc;
  int64_t ws_nrhs = 0;
};

namespace vsie {

int farnear_build(const vsie_mesh* near_m, int n_near, const vsie_mesh* far_m, int n_far, double freq, double tol,
                  const vsie_farnear_opts& o, vsie_farnear_s* h);
void farnear_entries(vsie_farnear_s* h, const int64_t* idx, int64_t count, void* out, cudaStream_t st);
void farnear_apply(vsie_farnear_s* h, const void* x, void* y, int op, int nrhs, cudaStream_t st);
void farnear_apply_pair(vsie_farnear_s* h, const void* x_far, void* y_near, const void* x_near, void* y_far,
                        cudaStream_t st);

}  // namespace vsie
