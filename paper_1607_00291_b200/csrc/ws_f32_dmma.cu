// Instantiations of the warp-specialised kernel: fp32 operands through DMMA (fp64 accumulation).
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_dmma(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_type<float, false>(a, stream);
}
}  // namespace tcb
