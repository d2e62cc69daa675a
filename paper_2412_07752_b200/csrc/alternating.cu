// alternating.cu -- per-step kernels for hidden sizes whose R exceeds on-chip
// capacity (placeholder until the streamed-R tcgen05 path lands).
#include "kernels.h"

namespace frnn {

size_t alt_forward_ws(const Problem&, const Plan&) { return 0; }
size_t alt_backward_ws(const Problem&, const Plan&) { return 0; }
cudaError_t alt_forward(const Problem&, const Plan&, void*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t alt_backward(const Problem&, const Plan&, void*, cudaStream_t) { return cudaErrorNotSupported; }

}  // namespace frnn
