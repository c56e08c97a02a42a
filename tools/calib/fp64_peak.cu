// FP64 peak calibration for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA throughput.
// Not part of the product path; used once per box to fix the roofline denominator
// (MEASURED_PEAKS.json has no FP64 figure).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dmma_m8n8k4_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_m16n8k16_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
double time_kernel(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(out, iters / 10);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_khz_attr\": %d}\n", p.name,
         p.multiProcessorCount, p.major, p.minor, clk_khz);
  double* out; CK(cudaMalloc(&out, 8));
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps, threads = wpb * 32;
      double ms = time_kernel(dmma_m8n8k4_loop<8>, blocks, threads, iters, out);
      double fl = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
      printf("{\"kind\": \"dmma_m8n8k4\", \"chains\": 8, \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, fl / ms / 1e9);
      ms = time_kernel(dmma_m16n8k16_loop<4>, blocks, threads, iters / 4, out);
      fl = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * blocks * wpb;
      printf("{\"kind\": \"dmma_m16n8k16\", \"chains\": 4, \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, fl / ms / 1e9);
      ms = time_kernel(dfma_loop<8>, blocks, threads, iters * 4, out);
      fl = 2.0 * 8 * (double)(iters * 4) * blocks * threads;
      printf("{\"kind\": \"dfma\", \"chains\": 8, \"warps_per_block\": %d, \"blocks\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             wpb, blocks, ms, fl / ms / 1e9);
    }
  }
  // DMMA latency probe: one chain, one warp
  {
    double ms = time_kernel(dmma_m8n8k4_loop<1>, 1, 32, iters, out);
    printf("{\"kind\": \"dmma_m8n8k4_latency\", \"ns_per_mma\": %.2f}\n", ms * 1e6 / iters);
  }
  return 0;
}
