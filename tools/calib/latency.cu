// Launch and memory-latency calibration for small contractions (cfg1 is an 18 us call):
// (1) empty kernel, 1 CTA x 384 threads, with 0 / 100 / 227 KB of dynamic shared memory;
// (2) one thread chasing a pointer chain through global memory (dependent loads), per load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu && ./latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* out) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && out) out[0] = s[0];
}

__global__ void chase(const long long* next, int steps, long long* out) {
  long long p = 0;
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  out[0] = p;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kb : {0, 100, 227}) {
    int smem = kb * 1024;
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int i = 0; i < 10; ++i) empty_kernel<<<1, 384, smem>>>(nullptr);
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) empty_kernel<<<1, 384, smem>>>(nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel, %3d KB smem: %.2f us per launch (back to back)\n", kb, 1e3f * ms / 200);
  }
  // pointer chase over 1 GiB (DRAM) and over 1 MiB (L2)
  for (size_t bytes : {(size_t)1 << 30, (size_t)1 << 20}) {
    size_t n = bytes / 8;
    long long* h = new long long[n];
    size_t stride = 4099 * 16;   // jump far enough to defeat sector reuse
    for (size_t i = 0; i < n; ++i) h[i] = (long long)((i + stride) % n);
    long long *d, *o;
    cudaMalloc(&d, bytes);
    cudaMalloc(&o, 8);
    cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(d, 1000, o);
    cudaEventRecord(e0);
    chase<<<1, 1>>>(d, 10000, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dependent load chain over %zu MiB: %.0f ns per load\n", bytes >> 20, 1e6f * ms / 10000);
    cudaFree(d);
    cudaFree(o);
    delete[] h;
  }
  return 0;
}
