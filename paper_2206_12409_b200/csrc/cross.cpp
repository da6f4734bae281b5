#include "cross.hpp"

namespace vsie {

int cross_build(vsie_coupling_s* h, double tol, const vsie_build_opts& o) {
  (void)h; (void)tol; (void)o;
  throw Error(VSIE_ERR_STATE, "cross_build: not implemented yet");
}

}  // namespace vsie
