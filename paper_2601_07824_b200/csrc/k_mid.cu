// k_mid.cu -- explicit instantiation of the single-pass kernels for N = 12..14 (k_mid).
#define SRE_FAMILY_MID
#include "launch.cuh"

namespace sre_host {
SRE_FOR_V_A2_DBG(SRE_SIG_MID, template);
}  // namespace sre_host
