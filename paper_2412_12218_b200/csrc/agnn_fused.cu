// Fused AGNN layer (placeholder until the single-pass kernel lands).
#include "kernels.cuh"

namespace sgtkcu {
void agnn_fused_launch(const sgtk_graph*, const float*, uint64_t, uint64_t, const float*, float,
                       int, float*, uint64_t, cudaStream_t) {
  raise(SGTK_ERR_RANGE, "agnn_forward: fused mode not available in this build");
}
}  // namespace sgtkcu
