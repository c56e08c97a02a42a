// Write patterns of a column-major C (ld = M = 15985, N = 16000 fp64: f1's k = 5 output) by CTA
// tiles of R rows x CB columns: which CTA -> region mapping streams C to HBM fastest. Each warp
// store is 32 consecutive rows (256 B) of one column. ORDER 0: blockIdx.x walks row blocks
// (fastest), 1: blockIdx.x walks column blocks. WALK > 0: grid.y = WALK CTAs per row block, each
// walking column blocks y, y + WALK, ... (the rank-k kernel's grid). Not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int R, int CB, int ORDER>
__global__ void __launch_bounds__(128) wp(double* __restrict__ C, int M, int N, int nrb, int ncb,
                                          int walk, double v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int rb, cb0, cstep;
  int cend = ncb;
  if (walk < 0) {   // ORDER 0 blocks, each CTA walking -walk consecutive column blocks
    rb = blockIdx.x % nrb; cb0 = (blockIdx.x / nrb) * -walk; cstep = 1;
    cend = min(ncb, cb0 - walk);
  } else if (walk > 0) { rb = blockIdx.x; cb0 = blockIdx.y; cstep = walk; }
  else if (ORDER == 0) { rb = blockIdx.x % nrb; cb0 = blockIdx.x / nrb; cstep = ncb; }
  else { cb0 = blockIdx.x % ncb; rb = blockIdx.x / ncb; cstep = ncb; }
  for (int cb = cb0; cb < cend; cb += cstep) {
#pragma unroll 4
    for (int j = warp; j < CB; j += 4) {
      const int c = cb * CB + j;
      if (c >= N) break;
#pragma unroll
      for (int r0 = 0; r0 < R; r0 += 32) {
        const int r = rb * R + r0 + lane;
        if (r < M) asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(C + (long long)c * M + r), "d"(v) : "memory");
      }
    }
  }
}

template <typename F>
float best(F f) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float m = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float t; CK(cudaEventElapsedTime(&t, a, b)); m = t < m ? t : m;
  }
  return m;
}

int main() {
  const int M = 15985, N = 16000;
  double* C; CK(cudaMalloc(&C, (size_t)M * N * 8));
  const double bytes = (double)M * N * 8;
#define P(R_, CB_, O_, WALK_) { const int nrb = (M + R_ - 1) / R_, ncb = (N + CB_ - 1) / CB_; \
    dim3 g = WALK_ > 0 ? dim3(nrb, WALK_) : WALK_ < 0 ? dim3((unsigned)(nrb * ((ncb - WALK_ - 1) / -WALK_))) : dim3((unsigned)(nrb * ncb)); \
    float ms = best([&] { wp<R_, CB_, O_><<<g, 128>>>(C, M, N, nrb, ncb, WALK_, 1.0); }); \
    printf("{\"R\": %d, \"CB\": %d, \"order\": %d, \"walk\": %d, \"gbs\": %.0f}\n", R_, CB_, O_, WALK_, bytes / ms / 1e6); }
  P(64, 32, 0, 38)     // the rank-k v2 grid: 250 row blocks x 38 = 64 CTAs per SM
  P(64, 32, 0, 0) P(128, 16, 0, 0) P(256, 16, 0, 0) P(256, 8, 0, 0)
  P(512, 4, 0, 0) P(512, 8, 0, 0) P(512, 16, 0, 0) P(1024, 4, 0, 0) P(1024, 8, 0, 0)
  P(2048, 2, 0, 0) P(2048, 4, 0, 0) P(4096, 2, 0, 0) P(16384, 1, 0, 0)
  P(512, 8, 0, -2) P(512, 8, 0, -4) P(512, 8, 0, -8) P(256, 16, 0, -4) P(1024, 8, 0, -4)
  P(64, 32, 0, -4) P(64, 32, 0, -16) P(256, 8, 0, -8)
  return 0;
}
