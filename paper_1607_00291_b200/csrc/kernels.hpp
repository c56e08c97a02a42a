// Device-side interface between tc_api.cpp and contract_kernels.cu.
#pragma once

#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace tcb {

// Tile shape of the sm_100a DMMA kernel. Tables are padded so that
// every tile-sized table read is in bounds.
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kBK = 16;
constexpr int kTablePad = 128;

// Launch arguments. All table pointers are device arrays of IDX (int32 or int64, per
// `idx64`), padded with zeros; vA / vB are block-scatter flags with block size 2 over the
// table that A / B is gathered along (1: the two entries are consecutive addresses).
struct LaunchArgs {
  const void* A;
  const void* B;
  void* C;
  const void* rA; const void* cA; const void* rB; const void* cB; const void* rC; const void* cC;
  const uint8_t* vA;
  const uint8_t* vB;
  int M, N, K;
  double alpha, beta;
  bool a_vec_m, b_vec_k, idx64, f32;
  // every pair of the operand's gather direction is contiguous and 16-byte aligned
  bool a_vec_all, b_vec_all;
  // fp32: every 8-byte pair of the operand's gather direction contiguous and 8-byte aligned
  bool a_vec2_all, b_vec2_all;
  // gather mode per operand (contract_ws.cuh GatherSel): 0 vectors, 1 per-vector check,
  // 2 coalesced elements; set by launch_contract from a_vec_all / b_vec_all and the plan
  int a_mode, b_mode;
  bool a_elem, b_elem;
  bool f32_a_transpose;
  bool c_lanes_n;
  int skinny_bu, skinny_bv;
  int tiny_mn_log2, tiny_mnk_log2;   // tiny.cu applies up to 2^mn elements of C, 2^mnk FMAs   // skinny kernel: X rows come in bv runs of bu (plan.cpp)        // FFMA epilogue: C's unit stride runs along N (lanes take columns)  // fp32 with A and B K-contiguous: transposing gather of A (mode 3)   // the plan prefers the element gather when not all vectors qualify
  // fp32, B gathered along N without aligned vectors: shifted 16-byte N vectors (umma_f32.cu
  // gather mode 12) through the per-tile-block run tables of tc_api.cpp nshift_tables:
  // bsh_p[tn][slot] = (block offset, run length and shift) pairs (int2), bsh_c[tn][n] = staging
  // word; b_shift: 0 = not available (no tables, B not 16-byte aligned, TC_UMMA_SHIFT=0),
  // 1 = available (the kernel decides), 2 = forced where available (TC_UMMA_SHIFT=2)
  const int* bsh_p;
  const int* bsh_c;
  int b_shift;
  int num_sms;        // persistent grid size (SMs of the current device)
  bool stream_k;      // split the final partial wave by K iterations
  bool f32_dmma;      // fp32 through the DMMA micro-kernel (fp64 accumulation) instead of FFMA
  int* flags;         // stream-K fix-up flags: >= flags_cap ints, private to the stream
  int flags_cap;      // flags[flags_cap] is the wave counter (monotonic, see Sched)
  // host copy of the stream's wave counter: a launch that aligns its waves takes its start
  // value and adds its whole tiles atomically (concurrent host threads on one stream)
  std::atomic<unsigned>* wave_base;
  unsigned flag_epoch;   // this launch's flag epoch, already shifted (epoch << 8, epoch >= 1)
  bool wave_sync;
};

// Skinny contractions (fp64, K <= 80, one free extent <= 96): skinny.cu.
// 0 = not applicable, 1 = launched, -1 = CUDA error.
// `force`: also when the streamed operand is not contiguous along its rows.
int launch_skinny(const LaunchArgs& a, cudaStream_t stream, bool force);

// Tiny contractions (<= 2^24 multiply-adds, <= 2^18 elements of C, K <= 256): tiny.cu, one
// thread per element of C. 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_tiny(const LaunchArgs& a, cudaStream_t stream);

// fp32 on the tcgen05 tensor cores with the 3xTF32 split: umma_f32.cu (int32 offsets, K >= 1).
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_umma_f32(const LaunchArgs& a, cudaStream_t stream);
int launch_umma_f32_n256(const LaunchArgs& a, cudaStream_t stream);   // element gathers only
int launch_umma_f32_pair(const LaunchArgs& a, cudaStream_t stream);   // CTA pairs (cta_group::2)
int launch_rankk(const LaunchArgs& a, cudaStream_t stream);   // K <= 16, large free extents

// Number of kernel launches it made, or -1 on a CUDA error (cudaGetLastError holds it).
int launch_contract(const LaunchArgs& a, cudaStream_t stream);

// The dynamic shared-memory opt-in (cudaFuncSetAttribute) applies to the kernel on the current
// device, so it is tracked per device (the largest size set so far); one process may drive
// several GPUs. Returns false on a CUDA error.
constexpr int kMaxDevices = 64;
template <typename K>
inline bool ensure_dyn_smem(K kern, int smem, std::atomic<int> (&done)[kMaxDevices]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return false;
  if (done[dev].load(std::memory_order_acquire) >= smem) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return false;
  int cur = done[dev].load(std::memory_order_relaxed);
  while (cur < smem && !done[dev].compare_exchange_weak(cur, smem, std::memory_order_release)) {
  }
  return true;
}

}  // namespace tcb
