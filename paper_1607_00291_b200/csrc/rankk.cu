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
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"

namespace tcb {
namespace rankk {

using namespace dev;

constexpr int kThreads = 128;   // 4 warps
constexpr int kRows = 64;       // rows of C per CTA (2 per lane)
constexpr int kNB = 32;         // columns per block (8 per warp)
constexpr int kMaxK = 8;
constexpr int kMaxK2 = 16;   // version 2 also takes 8 < K <= 16 (TC_RANKK16=1)
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

// Version 2 (default; TC_RANKK_V=1 selects the kernel above): the same grid (a CTA keeps one
// 64-row block and its A values in registers and walks column blocks y, y + gy, ...; CTAs
// resident together cover every row block of a few column blocks, so the stores of a wave fill
// a contiguous stretch of C), but the column blocks' C and B offsets and B values are staged with
// cp.async in rings, the offsets kD blocks before the values that use them (the values of block
// i + kD are gathered through offsets that landed with block i's group), so no thread waits on a
// dependent global load: version 1 stalled on its next block's two dependent loads (offsets,
// then values) at every block. One __syncthreads per block remains. Stores as in version 1.
#ifndef TC_RANKK_STNA
#define TC_RANKK_STNA 1   // C stores skip L1 allocation (st.global.L1::no_allocate)
#endif
constexpr int kD = 3;   // units of B values in flight (offsets: 2 kD + 1; rings of kD + 1 and 2 kD + 2)

template <typename T, typename IDX, int MAXK>
__global__ void __launch_bounds__(kThreads, MAXK <= 8 ? TC_RANKK_MINB : 4) tc_rankk2_kernel(Args p) {
  __shared__ __align__(16) T bs[kD + 1][MAXK][kNB];
  __shared__ IDX cy[2 * kD + 2][kNB];
  __shared__ IDX cs[2 * kD + 2][kNB];
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
  const int nblocks = (N + kNB - 1) / kNB;
  // this CTA's column blocks: blockIdx.y + i gridDim.y, i < nu
  // each CTA walks a consecutive range of column blocks: the CTAs resident together (all row
  // blocks of a few grid rows) then write few, long stretches of C, which HBM takes faster than
  // the interleaved stretches of a strided walk (f1 k = 5: 4.89 -> 5.16 TB/s;
  // profiles/r02/ab_rankk_walk.txt; tools/calib/write_pattern.cu). TC_RANKK_STRIDED (build
  // flag): the strided walk y, y + gy, ... of round 2's first version.
#ifdef TC_RANKK_STRIDED
  const int nu = blockIdx.y < nblocks ? (nblocks - 1 - (int)blockIdx.y) / (int)gridDim.y + 1 : 0;
  auto cb_of = [&](int i) { return (int)blockIdx.y + i * (int)gridDim.y; };
#else
  const int per = (nblocks + (int)gridDim.y - 1) / (int)gridDim.y;
  const int cb0 = (int)blockIdx.y * per;
  const int nu = cb0 < nblocks ? min(per, nblocks - cb0) : 0;
  auto cb_of = [&](int i) { return cb0 + i; };
#endif
  // the K offsets of Y, once
  IDX ky[MAXK];
#pragma unroll
  for (int k = 0; k < MAXK; ++k) ky[k] = k < K ? __ldg(kY + k) : 0;
  // stage the offsets of unit i (ring slot i % (2 kD + 1)): threads 0-31 cY, 32-63 cC
  auto stage_offsets = [&](int i) {
    if (i >= nu) return;
    const int n = cb_of(i) * kNB + (tid & 31);
    const int slot = i % (2 * kD + 2);
    if (tid < 32) {
      if constexpr (sizeof(IDX) == 8) cp_async8(&cy[slot][tid], cY + (n < N ? n : 0), n < N);
      else cp_async4(&cy[slot][tid], cY + (n < N ? n : 0), n < N);
    } else if (tid < 64) {
      if constexpr (sizeof(IDX) == 8) cp_async8(&cs[slot][tid - 32], cC + (n < N ? n : 0), n < N);
      else cp_async4(&cs[slot][tid - 32], cC + (n < N ? n : 0), n < N);
    }
  };
  // stage the B values of unit i (ring slot i % (kD + 1)) through its landed offsets
  auto stage_values = [&](int i) {
    if (i >= nu) return;
    const int n0 = cb_of(i) * kNB;
    const int oslot = i % (2 * kD + 2), vslot = i % (kD + 1);
    for (int e = tid; e < K * kNB; e += kThreads) {
      const int k = e / kNB, j = e - k * kNB;
      const bool in = n0 + j < N;
      const IDX o = in ? ky[0] : 0;
      IDX kk = 0;
#pragma unroll
      for (int q = 0; q < MAXK; ++q) kk = q == k ? ky[q] : kk;
      if constexpr (sizeof(T) == 8) cp_async8(&bs[vslot][k][j], Y + (in ? kk + cy[oslot][j] : o), in);
      else cp_async4(&bs[vslot][k][j], Y + (in ? kk + cy[oslot][j] : o), in);
    }
  };
  // prologue: offsets of units 0 .. 2kD-1 (groups 0 .. kD-1 carry two units each), then
  // values of units 0 .. kD-1 once their offsets have landed
  for (int g = 0; g < kD; ++g) {
    stage_offsets(2 * g);
    stage_offsets(2 * g + 1);
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int i = 0; i < kD; ++i) stage_values(i);
  stage_offsets(2 * kD);
  cp_async_commit();
  // (group accounting from here on: one group per unit i, holding the values of unit i + kD and
  //  the offsets of unit i + 2 kD + 1; the values of unit i are in the group of unit i - kD,
  //  or in the prologue group)
  // this CTA's rows and their K values of A, in registers for the whole kernel
  bool mv[2];
  IDX rc[2];
  double a[2][MAXK];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int m = (int)blockIdx.x * kRows + lane + 32 * h;
    mv[h] = m < M;
    const IDX rx = mv[h] ? rX[m] : 0;
    rc[h] = mv[h] ? rC[m] : 0;
#pragma unroll
    for (int k = 0; k < MAXK; ++k)
      a[h][k] = (mv[h] && k < K) ? static_cast<double>(X[rx + __ldg(kX + k)]) : 0.0;
  }
  for (int i = 0; i < nu; ++i) {
    const int cb = cb_of(i);
    cp_async_wait<kD - 1>();   // unit i's values (and unit i + kD's offsets) have landed
    __syncthreads();
    // refill: values of unit i + kD (offsets landed), offsets of unit i + 2 kD + 1
    stage_values(i + kD);
    stage_offsets(i + 2 * kD + 1);
    cp_async_commit();
    const int vslot = i % (kD + 1), oslot = i % (2 * kD + 2);
    double acc[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[h][j] = 0.0;
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      if (k < K) {
        double b[8];
        if constexpr (sizeof(T) == 8) {
          const double2* b2 = reinterpret_cast<const double2*>(&bs[vslot][k][8 * warp]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 v = b2[q];
            b[2 * q] = v.x;
            b[2 * q + 1] = v.y;
          }
        } else {
          const float4* b4 = reinterpret_cast<const float4*>(&bs[vslot][k][8 * warp]);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const float4 v = b4[q];
            b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[h][j] = fma(a[h][k], b[j], acc[h][j]);
      }
    }
    const int nw = cb * kNB + 8 * warp;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (nw + j < N) {
        const IDX cc = cs[oslot][8 * warp + j];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (mv[h]) {
            T* q = C + (rc[h] + cc);
            double v = p.alpha * acc[h][j];
            if (p.beta != 0.0) v = fma(p.beta, static_cast<double>(*q), v);
#if TC_RANKK_STNA
            st_na(q, static_cast<T>(v));
#else
            *q = static_cast<T>(v);
#endif
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <typename T, typename IDX>
static int launch_t(const Args& p, int num_sms, cudaStream_t s) {
  const int gx = (p.M + kRows - 1) / kRows;
  const int nblocks = (p.N + kNB - 1) / kNB;
  const char* v = getenv("TC_RANKK_V");
  const bool v1 = v && !strcmp(v, "1");
  // about TC_RANKK_OCC (version 2: TC_RANKK_OCC2) CTAs per SM in the grid; each walks its share
  // of the column blocks
  static const int occ2 = [] {
    const char* e = getenv("TC_RANKK_OCC2");
    return e ? atoi(e) : 64;
  }();
  long long gy = ((long long)(v1 ? TC_RANKK_OCC : occ2) * num_sms + gx - 1) / gx;
  if (gy > nblocks) gy = nblocks;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  if (v1) tc_rankk_kernel<T, IDX><<<dim3(gx, (unsigned)gy), kThreads, 0, s>>>(p);
  else if (p.K <= kMaxK) tc_rankk2_kernel<T, IDX, kMaxK><<<dim3(gx, (unsigned)gy), kThreads, 0, s>>>(p);
  else tc_rankk2_kernel<T, IDX, kMaxK2><<<dim3(gx, (unsigned)gy), kThreads, 0, s>>>(p);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace rankk

// Applies to 1 <= K <= 8 with at least 2^22 elements of C and both free extents >= 512.
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_rankk(const LaunchArgs& a, cudaStream_t stream) {
  const char* e16 = getenv("TC_RANKK16");   // read per call (tests switch it)
  const bool k16 = e16 && !strcmp(e16, "1");
  const char* v = getenv("TC_RANKK_V");
  const int maxk = (k16 && !(v && !strcmp(v, "1"))) ? rankk::kMaxK2 : rankk::kMaxK;
  if (a.K < 1 || a.K > maxk || a.M < 512 || a.N < 512 ||
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
