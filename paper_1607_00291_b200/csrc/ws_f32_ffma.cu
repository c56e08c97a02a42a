// Instantiations of the warp-specialised kernel: fp32 through the FFMA2 micro-kernel.
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_ffma(const LaunchArgs& a, cudaStream_t stream) {
  return ws::dispatch_type<float, true>(a, stream);
}
}  // namespace tcb
