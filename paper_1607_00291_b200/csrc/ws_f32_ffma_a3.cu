// Instantiations of the warp-specialised kernel: fp32 through the FFMA2 micro-kernel with A and
// B both gathered along K, A transposed into the [k][m] layout (gather mode 3).
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_ffma_a3(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_a_transposed<float, true>(a, stream);
}
}  // namespace tcb
