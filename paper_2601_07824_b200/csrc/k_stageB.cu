// k_stageB.cu -- explicit instantiation of the TMA-fed pass B of the staged and streamed paths.
#define SRE_FAMILY_STAGEB
#include "launch.cuh"

namespace sre_host {
SRE_FOR_V_A2(SRE_SIG_STAGEB, template);
}  // namespace sre_host
