// Tiny-contraction kernel (sm_100a): for contractions whose whole work is a few hundred
// thousand multiply-adds (BASELINE cfg1: abcd-aebf-dfce with all lengths 8, 64^3), the 128x128
// tensor-core tile would run on one SM and spend most of its time on padding. Here one thread
// computes one element of C directly from the definition through the scatter vectors
// (P:541-546): C[rC[m] + cC[n]] = alpha * sum_k A[rA[m] + cA[k]] * B[rB[k] + cB[n]] + beta * C,
// with an fp64 accumulator (rounded once for fp32, reading R12), spread over enough CTAs that
// the call costs little more than a launch.
#include <cstdint>

#include <cuda_runtime.h>

#include "kernels.hpp"

namespace tcb {
namespace tiny {

constexpr int kThreads = 128;   // consecutive m (C's unit-stride bundle)
// columns of C per thread (B shared through smem): 2 while the grid stays within four CTAs per
// SM, else 4 (cfg1 64^3: 5.3 -> 4.4 us; 512^2 x 64 prefers 4: 7.5 vs 10.9 us;
// profiles/r01/tiny_sweep_nb.txt)
constexpr int kNBMax = 4;
constexpr int kMaxK = 256;

// CTA = 128 consecutive rows x kNB columns of C. The CTA stages its kNB columns of B (K x kNB
// values) in shared memory; each thread loads A's values for its row kKB at a time into
// registers (K offsets read straight from the table: every lane reads the same entry, one
// broadcast), so a K loop of 64 costs two global round trips instead of eight, and the first
// block of A is already in flight while B is being staged. Each A value feeds kNB
// multiply-adds.
constexpr int kKB = 32;
template <typename T, typename IDX, int kNB>
__global__ void __launch_bounds__(kThreads) tc_tiny_kernel(
    const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
    const IDX* __restrict__ rA, const IDX* __restrict__ cA, const IDX* __restrict__ rB,
    const IDX* __restrict__ cB, const IDX* __restrict__ rC, const IDX* __restrict__ cC, int M,
    int N, int K, double alpha, double beta) {
  __shared__ double bs[kMaxK][kNB];
  const int m = blockIdx.x * kThreads + threadIdx.x;
  const int n0 = blockIdx.y * kNB;
  const bool mv = m < M;
  const IDX ra = mv ? rA[m] : 0;
  double a[kKB];
#pragma unroll
  for (int j = 0; j < kKB; ++j)
    a[j] = (mv && j < K) ? static_cast<double>(A[ra + __ldg(cA + j)]) : 0.0;
  for (int e = threadIdx.x; e < K * kNB; e += kThreads) {
    const int k = e / kNB, j = e - k * kNB;
    bs[k][j] = n0 + j < N ? static_cast<double>(B[rB[k] + cB[n0 + j]]) : 0.0;
  }
  __syncthreads();
  if (!mv) return;
  double acc[kNB];
#pragma unroll
  for (int j = 0; j < kNB; ++j) acc[j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kKB) {
    if (k0 > 0) {
#pragma unroll
      for (int j = 0; j < kKB; ++j)
        a[j] = k0 + j < K ? static_cast<double>(A[ra + __ldg(cA + k0 + j)]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kKB; ++j) {
      if (k0 + j < K) {
#pragma unroll
        for (int c = 0; c < kNB; ++c) acc[c] = fma(a[j], bs[k0 + j][c], acc[c]);
      }
    }
  }
  const IDX rc = rC[m];
#pragma unroll
  for (int j = 0; j < kNB; ++j) {
    if (n0 + j >= N) break;
    T* q = C + (rc + cC[n0 + j]);
    double v = alpha * acc[j];
    if (beta != 0.0) v = fma(beta, static_cast<double>(*q), v);
    *q = static_cast<T>(v);
  }
}

template <typename T, typename IDX, int kNB>
static int launch_nb(const LaunchArgs& a, cudaStream_t s) {
  const dim3 grid((a.M + kThreads - 1) / kThreads, (a.N + kNB - 1) / kNB);
  tc_tiny_kernel<T, IDX, kNB><<<grid, kThreads, 0, s>>>(
      static_cast<const T*>(a.A), static_cast<const T*>(a.B), static_cast<T*>(a.C),
      static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.M, a.N, a.K, a.alpha,
      a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T, typename IDX>
static int launch_t(const LaunchArgs& a, cudaStream_t s) {
  const long long ctas2 = (long long)((a.M + kThreads - 1) / kThreads) * ((a.N + 1) / 2);
  return ctas2 <= 4ll * a.num_sms ? launch_nb<T, IDX, 2>(a, s) : launch_nb<T, IDX, 4>(a, s);
}

}  // namespace tiny

// Applies when the contraction has at most 2^18 elements of C, at most 2^24 multiply-adds and
// K <= 256 (cfg1 is 2^12 / 2^18 / 64): there it beats the tensor-core tile kernel, whose few
// tiles run on few SMs (profiles/r01/tiny_sweep.jsonl, kernel time in CUDA graphs).
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_tiny(const LaunchArgs& a, cudaStream_t stream) {
  const long long mn = (long long)a.M * a.N;
  if (a.K > tiny::kMaxK || a.N > 65535 * tiny::kNBMax || mn > (1ll << a.tiny_mn_log2) ||
      mn * (a.K > 0 ? a.K : 1) > (1ll << a.tiny_mnk_log2))
    return 0;
  // fp32 hands the longer K loops to the tcgen05 kernel (256^3: 16 vs 22 us; 512^2 x 64 stays
  // here: 8.8 vs 25 us)
  if (a.f32 && a.K > 128) return 0;
  if (a.f32)
    return a.idx64 ? tiny::launch_t<float, long long>(a, stream)
                   : tiny::launch_t<float, int>(a, stream);
  return a.idx64 ? tiny::launch_t<double, long long>(a, stream)
                 : tiny::launch_t<double, int>(a, stream);
}

}  // namespace tcb
