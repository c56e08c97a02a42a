// Do DMMA (mma.sync f64) and DFMA share one FP64 datapath on B200? Warps 0..W/2-1 run DMMA
// chains, the others DFMA chains, in the same CTA; compare the combined rate with each alone.
// Not part of the product path (calibration for the skinny kernel's design).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// mode 0: all DMMA, 1: all DFMA, 2: half / half
template <int MODE>
__global__ void mix(double* out, int iters_mma, int iters_fma) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool do_mma = MODE == 0 || (MODE == 2 && warp < nw / 2);
  double s = 0;
  if (do_mma) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2] = {};
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
float run(int blocks, int threads, int im, int ifm, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  mix<MODE><<<blocks, threads>>>(out, im / 10, ifm / 10);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    mix<MODE><<<blocks, threads>>>(out, im, ifm);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  const int sms = 148, threads = 512, im = 20000;
  // per-warp flops: DMMA m8n8k4 = 512 flops x 8 chains per iter; DFMA = 32 x 2 x 8 per iter
  for (int ratio : {4, 8, 12}) {   // DFMA iterations per DMMA iteration (balances the halves)
    const int ifm = im * ratio;
    const double fm = 512.0 * 8 * im, ff = 64.0 * 8 * ifm;   // per warp
    const int nw = threads / 32;
    float t0 = run<0>(sms, threads, im, ifm, out);
    float t1 = run<1>(sms, threads, im, ifm, out);
    float t2 = run<2>(sms, threads, im, ifm, out);
    printf("{\"ratio\": %d, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"mixed_ms\": %.3f, "
           "\"mixed_tflops\": %.2f, \"dmma_alone_ms_half\": %.3f, \"dfma_alone_ms_half\": %.3f}\n",
           ratio, fm * nw * sms / t0 / 1e9, ff * nw * sms / t1 / 1e9, t2,
           (fm + ff) * (nw / 2) * sms / t2 / 1e9, t0 / 2, t1 / 2);
  }
  return 0;
}
