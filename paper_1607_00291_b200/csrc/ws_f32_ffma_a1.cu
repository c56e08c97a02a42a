// Instantiations of the warp-specialised kernel: fp32 through the FFMA2 micro-kernel, A gather mode 1
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_ffma_a1(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<float, true, 1>(a, stream);
}
int launch_ws_f32_ffma_idx64(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_idx64<float, true>(a, stream);
}
}  // namespace tcb
