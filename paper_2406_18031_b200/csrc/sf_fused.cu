// sf_fused.cu -- one-launch-per-frame fused predict + update (placeholder until the
// temporally blocked kernel lands; sf_step falls back to the per-pass kernels).
#include "sf_internal.cuh"

bool sf_fused_supported(const sf_ctx*) { return false; }
cudaError_t sf_launch_fused_step(sf_ctx*, const float*, const float*) { return cudaErrorNotSupported; }
int sf_fused_launches(const sf_ctx*) { return 0; }
