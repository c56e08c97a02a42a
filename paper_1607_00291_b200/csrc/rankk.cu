// Rank-k update kernel (sm_100a) for contractions whose bound extent K is at most 8 and whose
// free extents are large (m = n = 16000, k = 5): there the work is
// writing C (2 GB for fp64 at 16000^2) and the tensor-core tile spends most of its time on
// per-tile overheads, so this kernel is built around C's stores. A CTA owns 64 consecutive rows
// of C along its unit-stride bundle (lane l holds rows l and l + 32 with their K values of A in
// registers) and walks column blocks of 32; warp w forms columns 8w..8w+7 of a block, reading
// the block's K x 32 values of B from shared memory (double-buffered: the next block's loads
// are in flight while this one is stored) as 128-bit broadcasts. Every warp store is one
// 256-byte (fp64) run of C through its scatter vectors. When C's unit
// stride lies in the other free bundle the same kernel runs on the transposed problem
// (C^T = B^T A^T: the roles of the row and column tables swap), so the stores stay coalesced.
// Many small CTAs (TC_RANKK_OCC per SM in the grid) measured best (f1 k = 5: 8 per SM 0.93,
// 128 per SM 1.01 of DGEMM; adjacent-row vector stores 0.95, rejected;
// profiles/r01/ab_rankk.txt).
#include <cstdint>

#include <cuda_runtime.h>

#include "kernels.hpp"

namespace tcb {
namespace rankk {

constexpr int kThreads = 128;   // 4 warps
constexpr int kRows = 64;       // rows of C per CTA (2 per lane)
constexpr int kNB = 32;         // columns per block (8 per warp)
constexpr int kMaxK = 8;
#ifndef TC_RANKK_OCC
#define TC_RANKK_OCC 128
#endif

struct Args {
  const void* X;        // row operand: X[rX[m] + kX[k]]
  const void* Y;        // column operand: Y[kY[k] + cY[n]]
  void* C;              // C[rC[m] + cC[n]]
  const void *rX, *kX, *kY, *cY, *rC, *cC;
  int M, N, K;
  double alpha, beta;
};

#ifndef TC_RANKK_MINB
#define TC_RANKK_MINB 6   // six CTAs per SM (<= 85 registers): f1 k5 1.05 -> 1.11 of DGEMM
#endif
template <typename T, typename IDX>
__global__ void __launch_bounds__(kThreads, TC_RANKK_MINB) tc_rankk_kernel(Args p) {
  __shared__ __align__(16) double bs[2][kMaxK][kNB];
  __shared__ IDX cs[2][kNB];
  const T* __restrict__ X = static_cast<const T*>(p.X);
  const T* __restrict__ Y = static_cast<const T*>(p.Y);
  T* __restrict__ C = static_cast<T*>(p.C);
  const IDX* __restrict__ rX = static_cast<const IDX*>(p.rX);
  const IDX* __restrict__ kX = static_cast<const IDX*>(p.kX);
  const IDX* __restrict__ kY = static_cast<const IDX*>(p.kY);
  const IDX* __restrict__ cY = static_cast<const IDX*>(p.cY);
  const IDX* __restrict__ rC = static_cast<const IDX*>(p.rC);
  const IDX* __restrict__ cC = static_cast<const IDX*>(p.cC);
  const int M = p.M, N = p.N, K = p.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * kRows + lane;   // this lane's rows: m0, m0 + 32
  bool mv[2];
  IDX rc[2];
  double a[2][kMaxK];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = m0 + 32 * i;
    mv[i] = m < M;
    const IDX rx = mv[i] ? rX[m] : 0;
    rc[i] = mv[i] ? rC[m] : 0;
#pragma unroll
    for (int k = 0; k < kMaxK; ++k)
      a[i][k] = (mv[i] && k < K) ? static_cast<double>(X[rx + __ldg(kX + k)]) : 0.0;
  }
  const int nblocks = (N + kNB - 1) / kNB;
  auto stage = [&](int buf, int cb) {
    const int n0 = cb * kNB;
    for (int e = tid; e < K * kNB; e += kThreads) {
      const int k = e / kNB, j = e - k * kNB;
      bs[buf][k][j] = n0 + j < N ? static_cast<double>(Y[kY[k] + cY[n0 + j]]) : 0.0;
    }
    if (tid < kNB) cs[buf][tid] = n0 + tid < N ? cC[n0 + tid] : 0;
  };
  int buf = 0;
  int cb = blockIdx.y;
  if (cb < nblocks) stage(0, cb);
  __syncthreads();
  for (; cb < nblocks; cb += gridDim.y) {
    const int nxt = cb + gridDim.y;
    if (nxt < nblocks) stage(buf ^ 1, nxt);   // next block's loads overlap this block's stores
    double acc[2][8];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
      if (k < K) {
        const double2* b2 = reinterpret_cast<const double2*>(&bs[buf][k][8 * warp]);
        double b[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 v = b2[q];
          b[2 * q] = v.x;
          b[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i][k], b[j], acc[i][j]);
      }
    }
    const int nw = cb * kNB + 8 * warp;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (nw + j < N) {
        const IDX cc = cs[buf][8 * warp + j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (mv[i]) {
            T* q = C + (rc[i] + cc);
            double v = p.alpha * acc[i][j];
            if (p.beta != 0.0) v = fma(p.beta, static_cast<double>(*q), v);
            *q = static_cast<T>(v);
          }
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
}

template <typename T, typename IDX>
static int launch_t(const Args& p, int num_sms, cudaStream_t s) {
  const int gx = (p.M + kRows - 1) / kRows;
  const int nblocks = (p.N + kNB - 1) / kNB;
  // about TC_RANKK_OCC resident CTAs per SM; each walks its share of the column blocks
  long long gy = ((long long)TC_RANKK_OCC * num_sms + gx - 1) / gx;
  if (gy > nblocks) gy = nblocks;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  tc_rankk_kernel<T, IDX><<<dim3(gx, (unsigned)gy), kThreads, 0, s>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rankk

// Applies to 1 <= K <= 8 with at least 2^22 elements of C and both free extents >= 512.
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_rankk(const LaunchArgs& a, cudaStream_t stream) {
  if (a.K < 1 || a.K > rankk::kMaxK || a.M < 512 || a.N < 512 ||
      (long long)a.M * a.N < (1ll << 22))
    return 0;
  rankk::Args p;
  if (!a.c_lanes_n) {   // C's rows (M) hold its unit stride: rows = M
    p = {a.A, a.B, a.C, a.rA, a.cA, a.rB, a.cB, a.rC, a.cC, a.M, a.N, a.K, a.alpha, a.beta};
  } else {              // transposed problem: rows = N (B's columns), columns = M
    p = {a.B, a.A, a.C, a.cB, a.rB, a.cA, a.rA, a.cC, a.rC, a.N, a.M, a.K, a.alpha, a.beta};
  }
  if (a.f32)
    return a.idx64 ? rankk::launch_t<float, long long>(p, a.num_sms, stream)
                   : rankk::launch_t<float, int>(p, a.num_sms, stream);
  return a.idx64 ? rankk::launch_t<double, long long>(p, a.num_sms, stream)
                 : rankk::launch_t<double, int>(p, a.num_sms, stream);
}

}  // namespace tcb
