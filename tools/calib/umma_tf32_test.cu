// Standalone check of the tcgen05 kind::tf32 path (descriptors, TMEM, commit, tcgen05.ld):
// one CTA computes D[128 x 128] = A[128 x 32] . B[128 x 32]^T (K-major operands, SWIZZLE_NONE
// canonical layout) as plain TF32 and as 3xTF32 (hi.hi + hi.lo + lo.hi), compared on the host
// with an fp64 reference. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma umma_tf32_test.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int R = 128, KS = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major SWIZZLE_NONE descriptor: core matrices of 8 rows x 16 B; SBO = 8-row group stride,
// LBO = stride between the two 16-byte K halves of one 8-element tf32 MMA step.
__device__ __forceinline__ uint64_t make_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  return d;                  // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// element (r, k) of a 128 x 32 tile, in floats: K-major or MN-major canonical layout
template <bool MN>
__device__ __forceinline__ int tile_off(int r, int k) {
  return MN ? (k >> 3) * 1024 + (r >> 2) * 32 + (k & 7) * 4 + (r & 3)
            : (k >> 2) * (R * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

template <bool THREE, bool AMN, bool BMN>
__global__ void umma_test(const float* A, const float* B, float* D, uint32_t lbo_mn, uint32_t sbo_mn) {
  extern __shared__ __align__(1024) float dsm[];
  float* sa = dsm;
  float* sb = sa + R * KS;
  float* sal = sb + R * KS;
  float* sbl = sal + R * KS;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < R * KS; e += blockDim.x) {
    const int r = e / KS, k = e % KS;
    const float a = A[r * KS + k], b = B[r * KS + k];
    const float ah = THREE ? tf32_hi(a) : a, bh = THREE ? tf32_hi(b) : b;
    sa[tile_off<AMN>(r, k)] = ah;
    sb[tile_off<BMN>(r, k)] = bh;
    sal[tile_off<AMN>(r, k)] = a - ah;
    sbl[tile_off<BMN>(r, k)] = b - bh;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n"
                 :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) |
                         ((BMN ? 1u : 0u) << 16) | ((uint32_t)(R >> 3) << 17) |
                         ((uint32_t)(R >> 4) << 24);
  if (tid == 0) {
    const uint32_t LBO = R * 16, SBO = 128;
    for (int j = 0; j < KS / 8; ++j) {
      const int off = 2 * j * R * 4;   // floats: two 4-element K chunks per MMA step
      const float* ap[3] = {sa, sa, sal};
      const float* bp[3] = {sb, sbl, sb};
      for (int q = 0; q < (THREE ? 3 : 1); ++q) {
        const uint64_t da = AMN ? make_desc(ap[q] + off, lbo_mn, sbo_mn) : make_desc(ap[q] + off, LBO, SBO);
        const uint64_t db = BMN ? make_desc(bp[q] + off, lbo_mn, sbo_mn) : make_desc(bp[q] + off, LBO, SBO);
        const uint32_t acc = (j > 0 || q > 0) ? 1u : 0u;
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 :: "r"(smem_u32(&bar)) : "memory");
  }
  // wait for the MMAs (phase 0)
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n"
               :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < R; c0 += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 32; ++i) D[(32 * warp + lane) * R + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" :: "r"(tmem));
}

int main() {
  std::vector<float> A(R * KS), B(R * KS), D(R * R);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 4 * R * KS * 4;
  auto run = [&](auto kern, const char* name, uint32_t lbo, uint32_t sbo) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dD, 0, D.size() * 4);
    kern<<<1, 128, smem>>>(dA, dB, dD, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: CUDA error %s\n", name, cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (int m = 0; m < R; ++m)
      for (int n = 0; n < R; ++n) {
        double s = 0;
        for (int k = 0; k < KS; ++k) s += (double)A[m * KS + k] * B[n * KS + k];
        num += (D[m * R + n] - s) * (D[m * R + n] - s);
        den += s * s;
      }
    printf("%-28s lbo %5u sbo %5u: normwise rel err %.3e  D[0]=%f\n", name, lbo, sbo, sqrt(num / den), D[0]);
  };
  run(umma_test<false, false, false>, "TF32   K/K", 4096, 128);
  run(umma_test<true, false, false>, "3xTF32 K/K", 4096, 128);
  for (uint32_t lbo : {4096u, 128u}) for (uint32_t sbo : {128u, 4096u}) {
    run(umma_test<true, true, false>, "3xTF32 MN/K", lbo, sbo);
    run(umma_test<true, false, true>, "3xTF32 K/MN", lbo, sbo);
    run(umma_test<true, true, true>, "3xTF32 MN/MN", lbo, sbo);
  }
  return 0;
}
