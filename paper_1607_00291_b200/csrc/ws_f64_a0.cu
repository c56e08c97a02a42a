// Instantiations of the warp-specialised kernel: fp64 through the DMMA micro-kernel, A gather mode 0
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f64_a0(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<double, false, 0>(a, stream);
}
}  // namespace tcb
