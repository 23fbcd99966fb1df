// C ABI entry points that are not tied to one kernel family.
#include "mcf_internal.cuh"

namespace mcf {
const char *last_error();
}

extern "C" {

const char *mcf_version(void) { return "mcfunm_cuda 0.1.0 (sm_100a)"; }

const char *mcf_last_error(void) { return mcf::last_error(); }

}  // extern "C"
