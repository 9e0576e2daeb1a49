// attn_sm100.cu -- placeholder until the tcgen05 kernel lands.
#include "launch.cuh"
namespace sfa {
cudaError_t launch_attn_sm100(const AttnParams &, int, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace sfa
