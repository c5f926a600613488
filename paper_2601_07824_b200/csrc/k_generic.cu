// k_generic.cu -- explicit instantiation of the generic two-pass kernels (a < 2^L, unaligned heads, N = 26).
#define SRE_FAMILY_GENERIC
#include "launch.cuh"

namespace sre_host {
SRE_FOR_V(SRE_SIG_PASSA, template);
SRE_FOR_V_A2_DBG(SRE_SIG_PASSB, template);
}  // namespace sre_host
