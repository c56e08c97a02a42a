// st.async (register -> own CTA's shared memory, completion on an mbarrier with complete_tx)
// without a cluster launch: values land, the phase completes, no release fence needed by the
// storing thread (it keeps global loads in flight). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o st_async_test st_async_test.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t to_cluster(uint32_t a) {   // own CTA's address in the cluster window
  uint32_t r, rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__global__ void __cluster_dims__(1, 1, 1) k(const float* in, float* out, int iters) {
  __shared__ __align__(16) float buf[1024];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
  __syncthreads();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(4096));
    const float4 x = reinterpret_cast<const float4*>(in)[(it * 256 + threadIdx.x) % 4096];
    const uint32_t a = to_cluster((uint32_t)__cvta_generic_to_shared(buf + 4 * threadIdx.x));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(a), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w), "r"(to_cluster(b)) : "memory");
    asm volatile("{\n .reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 :: "r"(b), "r"(it & 1) : "memory");
    acc += buf[(threadIdx.x * 7) % 1024];
    __syncthreads();
  }
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main() {
  const int n = 4096 * 4, iters = 64;
  float *in, *out;
  cudaMalloc(&in, n * sizeof(float));
  cudaMalloc(&out, 256 * sizeof(float));
  float* h = new float[n];
  for (int i = 0; i < n; ++i) h[i] = (float)(i % 977);
  cudaMemcpy(in, h, n * sizeof(float), cudaMemcpyHostToDevice);
  k<<<1, 256>>>(in, out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  float o[256];
  cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int t = 0; t < 256; ++t) {
    float ref = 0.f;
    for (int it = 0; it < iters; ++it) {
      const int j = (t * 7) % 1024;             // element j of buf = float j % 4 of thread j / 4's vector
      const int src = ((it * 256 + j / 4) % 4096) * 4 + j % 4;
      ref += h[src];
    }
    bad += o[t] != ref;
  }
  printf("st.async test: %s, mismatches %d\n", cudaGetErrorString(e), bad);
  return bad != 0 || e != cudaSuccess;
}
