// Skinny-contraction kernel (sm_100a, fp64): one free bundle and the bound bundle are small
// (extent <= 96 and <= 80), the other free bundle is long -- e.g. fig:bench's abcde-efbad-cf
// with M ~ 1e6, N = K = 32. Such a contraction is an HBM stream: the long operand X
// (M x K) is read once and C (M x N) is written once, while the small operand Y (K x N) stays
// in shared memory for the whole kernel. The general 128 x 128 tile would spend most of its
// DMMA work on padding and restart its pipeline every 2-5 K steps.
//
// Persistent CTAs (one per SM, 256 threads) each load Y once (gathered through its scatter
// vectors), then walk 64-row blocks of X: a 3-deep ring of X blocks is gathered
// with cp.async (coalesced element copies along X's unit-stride direction, written to the
// [k][row] layout), each block is multiplied on the FP64 tensor cores (mma.sync m16n8k4 f64 ->
// DMMA.8x8x4; 8 warps = 4 row groups x 2 column halves) and written through the scatter
// vectors of C with alpha / beta (beta == 0 never reads C).
//
// Roles: X = A (rows = I, tables rA / cA), Y = B (cB / rB) when the small free bundle is J;
// X = B, Y = A (the transposed problem C^T = B^T A^T) when it is I.
#include <cstdint>
#include <cstdlib>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"

namespace tcb {
namespace skinny {

using namespace dev;

constexpr int kRows = 64;           // X rows per block
constexpr int kThreads = 256;
constexpr int kMaxN = 96;           // small free extent (padded to a multiple of 16)
constexpr int kMaxK = 80;           // bound extent (padded to a multiple of 4)
constexpr int kBufs = 3;            // X ring depth
constexpr int kXP = kRows + 4;      // [k][row] pitch (doubles): conflict-free fragment loads

struct Args {
  const double* X;
  const double* Y;
  double* C;
  const void* xr;   // X row table (long bundle)
  const void* xk;   // X K table
  const void* yk;   // Y K table
  const void* yc;   // Y column table (small bundle)
  const void* cr;   // C offsets along the long bundle
  const void* cc;   // C offsets along the small bundle
  int R, NC, K;     // long extent, small extent, bound extent
  int NP, KP;       // NC rounded up to 16, K rounded up to 4
  int bu, bv;       // X rows come in bv runs of bu contiguous elements (plan.cpp); 1, 1: plain
  double alpha, beta;
};

template <typename IDX, int NW>   // NW: n8 blocks per warp (NP / 16)
__device__ __forceinline__ void block_mma(const double* xs, const double* ys, int yp, int KP,
                                          int wr, int wc, int g, int t, double (&acc)[NW][4]) {
#pragma unroll
  for (int j = 0; j < NW; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = 0.0;
  // fragments of step k4 + 4 load while step k4 multiplies (KP is a multiple of 4)
  double a0 = xs[t * kXP + wr + g], a1 = xs[t * kXP + wr + g + 8], b[NW];
#pragma unroll
  for (int j = 0; j < NW; ++j) b[j] = ys[t * yp + wc + 8 * j + g];
  for (int k4 = 0; k4 < KP; k4 += 4) {
    const int kn = k4 + 4 < KP ? k4 + 4 : k4;
    const double na0 = xs[(kn + t) * kXP + wr + g], na1 = xs[(kn + t) * kXP + wr + g + 8];
    double nb[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) nb[j] = ys[(kn + t) * yp + wc + 8 * j + g];
#pragma unroll
    for (int j = 0; j < NW; ++j)
      dmma16x8x4(acc[j][0], acc[j][1], acc[j][2], acc[j][3], a0, a1, b[j]);
    a0 = na0; a1 = na1;
#pragma unroll
    for (int j = 0; j < NW; ++j) b[j] = nb[j];
  }
}

// ROWS_UNIT: X is contiguous along its rows (lanes take consecutive rows); otherwise along K
// (lanes take 8 consecutive K entries of 4 rows).
template <typename IDX, bool ROWS_UNIT, int NW, int kBufs>
__global__ void __launch_bounds__(kThreads, 1) tc_skinny_kernel(Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int yp = a.NP + 4;   // [k][col] pitch of Y (doubles), = 8 (mod 16) words per row
  double* ys = reinterpret_cast<double*>(smem_raw);
  double* xs = ys + a.KP * yp;
  // X's K offsets and C's small-bundle offsets, once per CTA (read from shared memory by the
  // loader and the epilogue instead of a dependent global load per copy / store)
  IDX* xks = reinterpret_cast<IDX*>(xs + kBufs * a.KP * kXP);
  IDX* ccs = xks + a.KP;
  const IDX* xr = static_cast<const IDX*>(a.xr);
  const IDX* xk = static_cast<const IDX*>(a.xk);
  const IDX* yk = static_cast<const IDX*>(a.yk);
  const IDX* yc = static_cast<const IDX*>(a.yc);
  const IDX* cr = static_cast<const IDX*>(a.cr);
  const IDX* cc = static_cast<const IDX*>(a.cc);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int k = tid; k < a.KP; k += kThreads) xks[k] = k < a.K ? xk[k] : 0;
  for (int n = tid; n < a.NP; n += kThreads) ccs[n] = n < a.NC ? cc[n] : 0;
  __syncthreads();
  // Y, once per CTA (zero-filled outside K x NC)
  for (int e = tid; e < a.KP * a.NP; e += kThreads) {
    const int k = e / a.NP, n = e - k * a.NP;
    const bool in = k < a.K && n < a.NC;
    cp_async8(ys + k * yp + n, a.Y + (in ? yk[k] + yc[n] : 0), in);
  }
  cp_async_commit();

  const int nblk = (a.R + kRows - 1) / kRows;
  // Per lane: two X rows of a block (rows-unit: rl[h] within the block; K-unit: 4 warp + 32 q
  // + (lane >> 3)). Their offsets are fetched one block ahead (rows()), so the loader never
  // waits on the row table when it issues the copies (issue()).
  const int bb = a.bu * a.bv;
  int rl[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if constexpr (ROWS_UNIT) {
      // with sub-divided rows, element e of the block is row (e % bu) bv + (e / bu) % bv +
      // (e / (bu bv)) bu bv, so consecutive lanes still read consecutive X elements
      const int e = 32 * h + lane;
      rl[h] = (e % a.bu) * a.bv + (e / a.bu) % a.bv + (e / bb) * bb;
    } else {
      rl[h] = 4 * warp + 32 * h + (lane >> 3);
    }
  }
  // (strides may be negative, so validity travels in rv, not in the offset)
  auto rows = [&](int blk, IDX (&ro)[2], bool (&rv)[2]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = blk * kRows + rl[h];
      rv[h] = blk < nblk && r < a.R;
      ro[h] = rv[h] ? xr[r] : 0;
    }
  };
  auto issue = [&](int buf, const IDX (&ro)[2], const bool (&rv)[2]) {
    double* d = xs + buf * (a.KP * kXP);
    if constexpr (ROWS_UNIT) {
#pragma unroll 4
      for (int k = warp; k < a.KP; k += kThreads / 32) {
        const bool kin = k < a.K;
        const IDX ko = xks[k];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          cp_async8(d + k * kXP + rl[h], a.X + (ro[h] + ko), kin && rv[h]);
      }
    } else {
      const int kk = lane & 7;
#pragma unroll 2
      for (int k0 = 0; k0 < a.KP; k0 += 8) {
        const int k = k0 + kk;
        if (k < a.KP) {
          const IDX ko = xks[k];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            cp_async8(d + k * kXP + rl[h], a.X + (ro[h] + ko), rv[h] && k < a.K);
        }
      }
    }
  };

  // ring of kBufs X blocks: blocks blockIdx.x + i * gridDim.x
  IDX ro[2];
  bool rv[2];
  for (int i = 0; i < kBufs - 1; ++i) {
    rows(blockIdx.x + i * gridDim.x, ro, rv);
    issue(i, ro, rv);
    cp_async_commit();
  }
  rows(blockIdx.x + (kBufs - 1) * gridDim.x, ro, rv);   // offsets of the next block to load
  const int g = lane >> 2, t = lane & 3;
  const int wr = 16 * (warp & 3), wc = (warp >> 2) * (a.NP / 2);
  double acc[NW][4];
  // C's row offsets of a block are fetched one block ahead as well
  auto crows = [&](int blk, IDX (&o)[2]) {
    const int r0 = blk * kRows + wr + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) o[h] = (blk < nblk && r0 + 8 * h < a.R) ? cr[r0 + 8 * h] : 0;
  };
  IDX cro[2], cro_next[2];
  crows(blockIdx.x, cro_next);
  for (int it = 0;; ++it) {
    const int blk = blockIdx.x + it * gridDim.x;
    if (blk >= nblk) break;
    const int cr0 = blk * kRows + wr + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) cro[h] = cro_next[h];
    crows(blk + gridDim.x, cro_next);
    // keep kBufs - 1 blocks in flight; prefetch the row offsets of the block after
    issue((it + kBufs - 1) % kBufs, ro, rv);
    cp_async_commit();
    rows(blockIdx.x + (it + kBufs) * gridDim.x, ro, rv);
    cp_async_wait<kBufs - 1>();
    __syncthreads();
    block_mma<IDX, NW>(xs + (it % kBufs) * (a.KP * kXP), ys, yp, a.KP, wr, wc, g, t, acc);
    // epilogue: rows wr + g (+8), columns wc + 8 j + 2 t (+1). A full block with every column
    // in range and beta == 0 stores without checks (the streaming case this kernel is for).
    if (a.beta == 0.0 && cr0 + 8 < a.R && a.NC == a.NP) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < NW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            a.C[cro[h] + ccs[wc + 8 * j + 2 * t + e]] = a.alpha * acc[j][2 * h + e];
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (cr0 + 8 * h >= a.R) continue;
#pragma unroll
        for (int j = 0; j < NW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = wc + 8 * j + 2 * t + e;
            if (n >= a.NC) continue;
            double* q = a.C + (cro[h] + ccs[n]);
            double v = a.alpha * acc[j][2 * h + e];
            if (a.beta != 0.0) v = fma(a.beta, *q, v);
            *q = v;
          }
      }
    }
    __syncthreads();   // the buffer of block `it` is refilled at iteration it + 1
  }
  cp_async_wait_all();
}

template <typename IDX, bool ROWS_UNIT, int NW, int NBUF>
static int launch_nb(const Args& a, int nsm, cudaStream_t s) {
  const int smem = (a.KP * (a.NP + 4) + NBUF * a.KP * kXP) * (int)sizeof(double) +
                   (a.KP + a.NP) * (int)sizeof(IDX);
  auto kern = tc_skinny_kernel<IDX, ROWS_UNIT, NW, NBUF>;
  static std::atomic<int> attr[kMaxDevices];
  if (!ensure_dyn_smem(kern, smem, attr)) return -1;
  const int nblk = (a.R + kRows - 1) / kRows;
  // low arithmetic intensity (small resident operand, e.g. N = K = 32: HBM-bound) runs four
  // CTAs per SM's worth of grid with a 2-deep ring, more CTAs in flight; larger ones one CTA with
  // a 3-deep ring (f2 strings: N = K = 32 0.88 -> 0.98 of DGEMM with three CTAs,
  // profiles/r01/ab_skinny_grid.txt; four CTAs x 2 buffers 3.34 -> 3.58 TB/s,
  // profiles/r02/ab_skinny_grid.txt; N = K = 76 -3..-5% with three)
  static const int cps_env = [] {   // measurement override (TC_SKINNY_CPS)
    const char* e = getenv("TC_SKINNY_CPS");
    return e ? atoi(e) : 0;
  }();
  const int cps = cps_env > 0 ? cps_env : (a.KP * a.NP <= 48 * 48 ? 4 : 1);
  const int grid = nblk < cps * nsm ? nblk : cps * nsm;
  kern<<<grid, kThreads, smem, s>>>(a);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Ring depth 3 (kBufs). A 6-deep ring, for more bytes in flight per SM, measured slower on
// the HBM-bound f2 strings (0.84 -> 0.64 of DGEMM).
template <typename IDX, bool ROWS_UNIT, int NW>
static int launch_nw(const Args& a, int nsm, cudaStream_t s) {
  static const int nbuf_env = [] {   // measurement override (TC_SKINNY_NBUF = 2 | 3 | 4)
    const char* e = getenv("TC_SKINNY_NBUF");
    return e ? atoi(e) : 0;
  }();
  const int nbuf = nbuf_env > 0 ? nbuf_env : (a.KP * a.NP <= 48 * 48 ? 2 : kBufs);
  if (nbuf == 2) return launch_nb<IDX, ROWS_UNIT, NW, 2>(a, nsm, s);
  if (nbuf == 4) return launch_nb<IDX, ROWS_UNIT, NW, 4>(a, nsm, s);
  return launch_nb<IDX, ROWS_UNIT, NW, kBufs>(a, nsm, s);
}

template <typename IDX, bool ROWS_UNIT>
static int launch_dir(const Args& a, int nsm, cudaStream_t s) {
  switch (a.NP / 16) {
    case 1: return launch_nw<IDX, ROWS_UNIT, 1>(a, nsm, s);
    case 2: return launch_nw<IDX, ROWS_UNIT, 2>(a, nsm, s);
    case 3: return launch_nw<IDX, ROWS_UNIT, 3>(a, nsm, s);
    case 4: return launch_nw<IDX, ROWS_UNIT, 4>(a, nsm, s);
    case 5: return launch_nw<IDX, ROWS_UNIT, 5>(a, nsm, s);
    default: return launch_nw<IDX, ROWS_UNIT, 6>(a, nsm, s);
  }
}

}  // namespace skinny

// The skinny path applies to fp64 contractions with K <= 80 and one free extent <= 96 (the
// small extent becomes the resident operand's columns). `force` = false restricts it to a
// streamed operand that is contiguous along the long bundle (launch_contract passes true unless
// TC_SKINNY=0 turns the path off). Returns 0 when it does not apply, 1 on launch, -1 on a CUDA
// error.
int launch_skinny(const LaunchArgs& la, cudaStream_t stream, bool force) {
  using namespace skinny;
  if (la.f32 || la.K < 1 || la.K > kMaxK) return 0;
  const bool small_n = la.N <= kMaxN;
  const bool small_m = !small_n && la.M <= kMaxN;
  if (!small_n && !small_m) return 0;
  Args a{};
  bool rows_unit;
  if (small_n) {   // X = A (rows M), Y = B
    a.X = static_cast<const double*>(la.A); a.Y = static_cast<const double*>(la.B);
    a.xr = la.rA; a.xk = la.cA; a.yk = la.rB; a.yc = la.cB; a.cr = la.rC; a.cc = la.cC;
    a.R = la.M; a.NC = la.N;
    rows_unit = la.a_vec_m;
  } else {         // X = B (rows N), Y = A: C^T = B^T A^T
    a.X = static_cast<const double*>(la.B); a.Y = static_cast<const double*>(la.A);
    a.xr = la.cB; a.xk = la.rB; a.yk = la.cA; a.yc = la.rA; a.cr = la.cC; a.cc = la.rC;
    a.R = la.N; a.NC = la.M;
    rows_unit = !la.b_vec_k;
  }
  if (!rows_unit && !force) return 0;
  a.C = static_cast<double*>(la.C);
  a.K = la.K;
  a.NP = (a.NC + 15) / 16 * 16;
  a.KP = (a.K + 3) / 4 * 4;
  a.alpha = la.alpha; a.beta = la.beta;
  a.bu = la.skinny_bu > 0 ? la.skinny_bu : 1;
  a.bv = la.skinny_bv > 0 ? la.skinny_bv : 1;
  if (la.idx64)
    return rows_unit ? launch_dir<long long, true>(a, la.num_sms, stream)
                     : launch_dir<long long, false>(a, la.num_sms, stream);
  return rows_unit ? launch_dir<int, true>(a, la.num_sms, stream)
                   : launch_dir<int, false>(a, la.num_sms, stream);
}

}  // namespace tcb
