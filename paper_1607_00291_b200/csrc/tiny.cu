// Tiny-contraction kernel (sm_100a): for contractions whose whole work is a few hundred
// thousand multiply-adds (BASELINE cfg1: abcd-aebf-dfce with all lengths 8, 64^3), the 128x128
// tensor-core tile would run on one SM and spend most of its time on padding. Here one thread
// computes one element of C directly from the definition through the scatter vectors
// (P:541-546): C[rC[m] + cC[n]] = alpha * sum_k A[rA[m] + cA[k]] * B[rB[k] + cB[n]] + beta * C,
// with an fp64 accumulator (rounded once for fp32, reading R12), spread over enough CTAs that
// the call costs little more than a launch. Threads run along M so that C's unit-stride
// bundle (put first by the heuristic) is written by consecutive lanes.
#include <cstdint>

#include <cuda_runtime.h>

#include "kernels.hpp"

namespace tcb {
namespace tiny {

constexpr int kThreads = 128;

template <typename T, typename IDX>
__global__ void __launch_bounds__(kThreads) tc_tiny_kernel(
    const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
    const IDX* __restrict__ rA, const IDX* __restrict__ cA, const IDX* __restrict__ rB,
    const IDX* __restrict__ cB, const IDX* __restrict__ rC, const IDX* __restrict__ cC, int M,
    int N, int K, double alpha, double beta) {
  const long long e = (long long)blockIdx.x * kThreads + threadIdx.x;
  if (e >= (long long)M * N) return;
  const int m = (int)(e % M), n = (int)(e / M);
  const IDX ra = rA[m], cb = cB[n];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // four partial sums: independent FMAs
  int k = 0;
  for (; k + 4 <= K; k += 4) {
    s0 = fma(static_cast<double>(A[ra + cA[k]]), static_cast<double>(B[rB[k] + cb]), s0);
    s1 = fma(static_cast<double>(A[ra + cA[k + 1]]), static_cast<double>(B[rB[k + 1] + cb]), s1);
    s2 = fma(static_cast<double>(A[ra + cA[k + 2]]), static_cast<double>(B[rB[k + 2] + cb]), s2);
    s3 = fma(static_cast<double>(A[ra + cA[k + 3]]), static_cast<double>(B[rB[k + 3] + cb]), s3);
  }
  for (; k < K; ++k)
    s0 = fma(static_cast<double>(A[ra + cA[k]]), static_cast<double>(B[rB[k] + cb]), s0);
  T* q = C + (rC[m] + cC[n]);
  double v = alpha * ((s0 + s1) + (s2 + s3));
  if (beta != 0.0) v = fma(beta, static_cast<double>(*q), v);
  *q = static_cast<T>(v);
}

template <typename T, typename IDX>
static int launch_t(const LaunchArgs& a, cudaStream_t s) {
  const long long n = (long long)a.M * a.N;
  const int grid = (int)((n + kThreads - 1) / kThreads);
  tc_tiny_kernel<T, IDX><<<grid, kThreads, 0, s>>>(
      static_cast<const T*>(a.A), static_cast<const T*>(a.B), static_cast<T*>(a.C),
      static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.M, a.N, a.K, a.alpha,
      a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace tiny

// Applies when the whole contraction is at most 2^21 multiply-adds over at most 2^16 elements
// of C (cfg1 is 2^18 over 2^12). 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_tiny(const LaunchArgs& a, cudaStream_t stream) {
  const long long mn = (long long)a.M * a.N;
  if (mn > (1ll << 16) || mn * (a.K > 0 ? a.K : 1) > (1ll << 21)) return 0;
  if (a.f32)
    return a.idx64 ? tiny::launch_t<float, long long>(a, stream)
                   : tiny::launch_t<float, int>(a, stream);
  return a.idx64 ? tiny::launch_t<double, long long>(a, stream)
                 : tiny::launch_t<double, int>(a, stream);
}

}  // namespace tcb
