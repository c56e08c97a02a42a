// tcgen05.mma kind::tf32 issue rate on one SM: a single thread issues R rounds of 12 MMAs
// (M = N = 128, K = 8; A from TMEM or shared memory, B from shared memory) into one TMEM
// accumulator, committing to an mbarrier every round and waiting `lag` rounds behind; the
// elapsed clock64 cycles per MMA against the nominal 65 cycles (1.125 PF/s dense TF32 / 148 SMs
// / 1.9 GHz = 4000 flop/cycle, 262144 flop per MMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate_test.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void rate(int rounds, int a_tmem, int n256, int alt, long long* out) {
  extern __shared__ __align__(1024) float sm[];   // A 128 x 32, B 256 x 32 (contents irrelevant)
  __shared__ __align__(8) uint64_t bar[2];   // alternating: a barrier completes once per check
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * 128 * 32; i += blockDim.x) sm[i] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0)
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bar[b])));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((n256 ? 32u : 16u) << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      for (int q = 0; q < 3; ++q)
        for (int j = 0; j < 4; ++j) {
          const uint32_t dst = tmem + (uint32_t)(alt == 1 ? ((q * 4 + j) & 1) * 128
                                                 : alt == 2 ? (r & 1) * 128 : 0);
          const uint64_t db = make_desc(sm + 128 * 32 + j * 2048, n256 ? 4096 : 2048, 128);
          if (a_tmem) {
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                         :: "r"(dst), "r"(tmem + 256 + 8 * j), "l"(db), "r"(idesc), "r"(1));
          } else {
            const uint64_t da = make_desc(sm + j * 1024, 2048, 128);
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                         " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(dst), "l"(da), "l"(db), "r"(idesc), "r"(1));
          }
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                   :: "r"(smem_u32(&bar[r & 1])) : "memory");
      // wait for the previous round's commit (one round in flight)
      if (r > 0) {
        const int q = r - 1;
        asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                     :: "r"(smem_u32(&bar[q & 1])), "r"((q >> 1) & 1) : "memory");
      }
    }
    {
      const int q = rounds - 1;
      asm volatile("{\n .reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2;\n}\n"
                   :: "r"(smem_u32(&bar[q & 1])), "r"((q >> 1) & 1) : "memory");
    }
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tmem));
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  const int smem = 3 * 128 * 32 * 4;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v = 0; v < 7; ++v) {
    const int a_tmem = v < 4 ? (v & 1) : 1, n256 = v < 4 ? v >> 1 : 0, alt = v < 4 ? 0 : v - 3;
    if (alt == 3) {   // N = 256 from smem with per-round alternation would need 512 + A: skip
      continue;
    }
    const int rounds = 2000;
    rate<<<1, 128, smem>>>(rounds, a_tmem, n256, alt, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N = %d, A from %s, accumulators %s: %.1f cycles per 128x%dx8 tf32 MMA (nominal %d)\n",
           n256 ? 256 : 128, a_tmem ? "TMEM" : "smem",
           alt == 0 ? "one" : alt == 1 ? "two, alternating per MMA" : "two, alternating per round",
           (double)c / (rounds * 12.0), n256 ? 256 : 128, n256 ? 131 : 65);
  }
  return 0;
}
