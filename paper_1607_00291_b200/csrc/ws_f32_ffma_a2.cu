// Instantiations of the warp-specialised kernel: fp32 through the FFMA2 micro-kernel, A gather mode 2
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_ffma_a2(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<float, true, 2>(a, stream);
}
}  // namespace tcb
