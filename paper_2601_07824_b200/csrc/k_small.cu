// k_small.cu -- explicit instantiation of the single-pass kernels for N <= 11 (k_small).
#define SRE_FAMILY_SMALL
#include "launch.cuh"

namespace sre_host {
SRE_FOR_V_A2_DBG(SRE_SIG_SMALL, template);
}  // namespace sre_host
