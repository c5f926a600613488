// k_stageA.cu -- explicit instantiation of the pass A of the staged (N = 15..20) and streamed (N = 21..25) paths.
#define SRE_FAMILY_STAGEA
#include "launch.cuh"

namespace sre_host {
SRE_FOR_V(SRE_SIG_STAGEA, template);
}  // namespace sre_host
