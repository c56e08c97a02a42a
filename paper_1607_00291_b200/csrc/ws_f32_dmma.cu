// Instantiations of the warp-specialised kernel: fp32 operands through DMMA (fp64 accumulation;
// TC_F32_MMA=dmma ablation). Per-vector gathers only (modes 0 and 1).
#include "contract_ws.cuh"

namespace tcb {
int launch_ws_f32_dmma(const LaunchArgs& a, cudaStream_t stream) {
  if (a.idx64) return ws::dispatch_idx64<float, false>(a, stream);
  const int am = a.a_mode == 0 ? 0 : 1, bm = a.b_mode == 0 ? 0 : 1;
  if (am == 0)
    return bm == 0 ? ws::dispatch_dir<float, int, 0, 0, false>(a, stream)
                   : ws::dispatch_dir<float, int, 0, 1, false>(a, stream);
  return bm == 0 ? ws::dispatch_dir<float, int, 1, 0, false>(a, stream)
                 : ws::dispatch_dir<float, int, 1, 1, false>(a, stream);
}
}  // namespace tcb
