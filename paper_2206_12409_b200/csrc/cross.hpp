// DMRG two-site TT-cross driver.
#pragma once

#include "handle.hpp"

namespace vsie {

// Builds the three chi TTs of the handle's Z_bc by TT-cross over the entry
// kernel.  Returns VSIE_OK or VSIE_WARN_NOT_CONVERGED; throws on errors.
int cross_build(vsie_coupling_s* h, double tol, const vsie_build_opts& o);

// TT rounding (recompression) of the handle's cores in place, relative Frobenius
// accuracy tol per chi (algorithm in cross.cpp).  World 1 / loopback.
int tt_round(vsie_coupling_s* h, double tol);

}  // namespace vsie
