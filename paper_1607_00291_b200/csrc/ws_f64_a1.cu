// Instantiations of the warp-specialised kernel: fp64 through the DMMA micro-kernel, A gather mode 1
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f64_a1(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<double, false, 1>(a, stream);
}
int launch_ws_f64_idx64(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_idx64<double, false>(a, stream);
}
}  // namespace tcb
