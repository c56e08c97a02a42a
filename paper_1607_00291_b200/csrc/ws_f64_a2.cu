// Instantiations of the warp-specialised kernel: fp64 through the DMMA micro-kernel, A gather mode 2
// (contract_ws.cuh GatherSel), every B gather mode and loader direction.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f64_a2(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_b<double, false, 2>(a, stream);
}
}  // namespace tcb
