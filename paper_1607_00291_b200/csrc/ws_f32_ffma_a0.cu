// Instantiations of the warp-specialised kernel: fp32 through the FFMA2 micro-kernel, A gather mode 0
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_ffma_a0(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<float, true, 0>(a, stream);
}
}  // namespace tcb
