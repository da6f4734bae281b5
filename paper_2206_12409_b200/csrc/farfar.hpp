// Dense far-far conductor block (farfar.cu): the handle behind include/vsie_farfar.h.
#pragma once

#include "../../include/vsie_farfar.h"
#include "kernels.cuh"

struct vsie_farfar_s {
  int device = 0;
  int64_t m = 0, nt = 0;        // RWG functions, triangles
  int nb = 0;                   // 128-blocks
  int64_t tiles = 0, near_pairs = 0, apply_calls = 0;
  double k0 = 0, build_s = 0, scale_re = 1, scale_im = 0;
  vsie::DevBuf<double> tri;     // [nt][32] per triangle: V[9], centroid[3], normal[3], nodes[9], A, L
  vsie::DevBuf<int> rt;         // [m][2] T+ / T- triangle ids
  vsie::DevBuf<double> rp;      // [m][8] p+[3], p-[3], l
  vsie::DevBuf<vsie::cplx> Z;   // tiles
  vsie::DevBuf<vsie::cplx> part;   // [tiles][256] apply partials
  vsie::DevBuf<vsie::cplx> xc;     // OP_C conj(x) scratch [m]
};

namespace vsie {

void farfar_build(const vsie_mesh* meshes, int n_meshes, double freq, double scale_re, double scale_im, int device,
                  vsie_farfar_s* h);
void farfar_entries(vsie_farfar_s* h, const int64_t* idx, int64_t count, void* out, cudaStream_t st);
void farfar_apply(vsie_farfar_s* h, const void* x, void* y, int op, int nrhs, bool accumulate, cudaStream_t st);
void farfar_export(vsie_farfar_s* h, void* host_dense);

}  // namespace vsie
