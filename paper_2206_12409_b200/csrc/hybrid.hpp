// The GMRES consumer of the hybrid VSIE system (hybrid.cu): internal entry points behind
// include/vsie_hybrid.h.
#pragma once

#include "../../include/vsie_hybrid.h"
#include "kernels.cuh"

struct vsie_farfar_s;
struct vsie_farnear_s;
struct vsie_coupling_s;

namespace vsie {

vsie_hybrid_s* hybrid_new();
void hybrid_delete(vsie_hybrid_s* h);
void hybrid_create(vsie_farfar_s* ff, vsie_farnear_s* fn, vsie_farfar_s* nn, vsie_coupling_s* cbf,
                   vsie_coupling_s* cbn, const void* d_body, vsie_hybrid_s* h);
void hybrid_matvec(vsie_hybrid_s* h, const void* x, void* y, cudaStream_t st);
int hybrid_gmres(vsie_hybrid_s* h, const void* b, void* x, int restart, int max_iter, double tol, double* history,
                 vsie_gmres_info* info, cudaStream_t st);
void hybrid_info(vsie_hybrid_s* h, vsie_hybrid_info* out);

}  // namespace vsie
