// Instantiations of the warp-specialised kernel: fp64 (DMMA).
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f64(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_type<double, false>(a, stream);
}
}  // namespace tcb
