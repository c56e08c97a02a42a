// Skinny-contraction kernel (sm_100a, fp64): one free bundle and the bound bundle are small
// (extent <= 96 and <= 80), the other free bundle is long -- e.g. fig:bench's abcde-efbad-cf
// with M ~ 1e6, N = K = 32. Such a contraction is an HBM stream: the long operand X
// (M x K) is read once and C (M x N) is written once, while the small operand Y (K x N) stays
// in shared memory for the whole kernel. The general 128 x 128 tile would spend most of its
// DMMA work on padding and restart its pipeline every 2-5 K steps.
//
// Two forms. The default is warp-specialised (tc_skinny_ws_kernel below: producer warps, an
// mbarrier ring, consumer warps; Y in registers for N, K <= 32). The synchronous form (kept for
// TC_SKINNY_WS=0 and as the fallback when the ring does not fit):
// Persistent CTAs (256 threads) each load Y once (gathered through its scatter
// vectors), then walk 64-row blocks of X: a 2-3-deep ring of X blocks is gathered
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
constexpr int kXPSkew = kRows + 20; // pitch with a skewed row layout (Args::sw > 0), = 4 (mod 16)

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
  int xp, sw;       // X ring pitch (doubles) and row skew: block row r sits at r + sw (r / 16)
  int dbg;          // measurement only (TC_SKINNY_DBG): 1 skip the MMA, 2 the X loads, 4 the stores
  double alpha, beta;
};

// wr: the warp's first row position in the ring buffer (16 rows, contiguous), xp its pitch
template <typename IDX, int NW>   // NW: n8 blocks per warp (NP / 16)
__device__ __forceinline__ void block_mma(const double* xs, int xp, const double* ys, int yp,
                                          int KP, int wr, int wc, int g, int t,
                                          double (&acc)[NW][4]) {
#pragma unroll
  for (int j = 0; j < NW; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = 0.0;
  // fragments of step k4 + 4 load while step k4 multiplies (KP is a multiple of 4)
  double a0 = xs[t * xp + wr + g], a1 = xs[t * xp + wr + g + 8], b[NW];
#pragma unroll
  for (int j = 0; j < NW; ++j) b[j] = ys[t * yp + wc + 8 * j + g];
  for (int k4 = 0; k4 < KP; k4 += 4) {
    const int kn = k4 + 4 < KP ? k4 + 4 : k4;
    const double na0 = xs[(kn + t) * xp + wr + g], na1 = xs[(kn + t) * xp + wr + g + 8];
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
#ifndef TC_SKINNY_MINB
#define TC_SKINNY_MINB 1   // experiment: -DTC_SKINNY_MINB=3 caps registers for 3 CTAs per SM
#endif
template <typename IDX, bool ROWS_UNIT, int NW, int kBufs>
__global__ void __launch_bounds__(kThreads, TC_SKINNY_MINB) tc_skinny_kernel(Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int yp = a.NP + 4;   // [k][col] pitch of Y (doubles), = 8 (mod 16) words per row
  double* ys = reinterpret_cast<double*>(smem_raw);
  double* xs = ys + a.KP * yp;
  // X's K offsets and C's small-bundle offsets, once per CTA (read from shared memory by the
  // loader and the epilogue instead of a dependent global load per copy / store)
  const int xp = a.xp;
  IDX* xks = reinterpret_cast<IDX*>(xs + kBufs * a.KP * xp);
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
  int rl[2], pl[2];   // block row, and its position in the ring buffer (skewed)
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
    pl[h] = rl[h] + a.sw * (rl[h] >> 4);
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
    if (a.dbg & 2) return;
    double* d = xs + buf * (a.KP * xp);
    if constexpr (ROWS_UNIT) {
#pragma unroll 4
      for (int k = warp; k < a.KP; k += kThreads / 32) {
        const bool kin = k < a.K;
        const IDX ko = xks[k];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          cp_async8(d + k * xp + pl[h], a.X + (ro[h] + ko), kin && rv[h]);
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
            cp_async8(d + k * xp + pl[h], a.X + (ro[h] + ko), rv[h] && k < a.K);
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
    if (!(a.dbg & 1)) {
      block_mma<IDX, NW>(xs + (it % kBufs) * (a.KP * xp), xp, ys, yp, a.KP,
                         wr + a.sw * (wr >> 4), wc, g, t, acc);
    } else {
#pragma unroll
      for (int j = 0; j < NW; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[j][q] = xs[(it % kBufs) * (a.KP * xp) + q * xp + wr + g];
    }
    if (a.dbg & 4) { __syncthreads(); continue; }
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
  const int smem = (a.KP * (a.NP + 4) + NBUF * a.KP * a.xp) * (int)sizeof(double) +
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

// ---- warp-specialised form (the HBM-bound class: NP <= 32, KP <= 32) -------------------------
// The synchronous kernel above loads a block, waits, multiplies, stores: per SM at most two
// blocks are in flight and the DMMA pipe idles while a CTA waits (f2_00: X loads alone 66 us,
// stores alone 81 us, MMA alone 83 us, all three 137 us; profiles/r02/ab_skinny_ws.txt). Here one
// persistent CTA per SM splits the roles: kWsProd producer warps gather X blocks into an S-deep
// ring (cp.async, completion tracked by an mbarrier per stage), and CG groups of 8 consumer warps
// multiply (Y held in registers for the CTA's lifetime), release the stage, and store C from
// registers. Up to S - 1 blocks per SM are in flight while the consumers compute.
constexpr int kWsProd = 4;
// (larger resident operands, Y from shared memory, one consumer group: the N = K = 76 strings
//  f2_02/04/06/12/13/14 1.06-1.18 -> 1.11-1.31 of DGEMM)
constexpr int kWsMaxK4 = 8;   // KP <= 32
constexpr int kWsAhead = 4;   // producer: row-offset lookahead (blocks)

// X copies of the warp-specialised producers: 8-byte cp.async, optionally with an L2 prefetch
// hint (TC_SKINNY_L2HINT = 128 | 256 build flag, measurement; profiles/r02/ab_skinny_l2hint.txt)
#ifndef TC_SKINNY_L2HINT
#define TC_SKINNY_L2HINT 0
#endif
__device__ __forceinline__ void cp_async8_x(void* smem, const void* gmem, bool pred) {
  const int sz = pred ? 8 : 0;
  if constexpr (TC_SKINNY_L2HINT == 256)
    asm volatile("cp.async.ca.shared.global.L2::256B [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(sz));
  else if constexpr (TC_SKINNY_L2HINT == 128)
    asm volatile("cp.async.ca.shared.global.L2::128B [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(sz));
  else
    cp_async8(smem, gmem, pred);
}

// YREG: Y's fragments live in registers (NP, KP <= 32); otherwise the consumers read them from
// shared memory per block (block_mma), for the larger resident operands (K, N <= 80, 96).
template <typename IDX, bool ROWS_UNIT, int NW, int CG, bool YREG>
__global__ void __launch_bounds__(32 * (kWsProd + 8 * CG), 1) tc_skinny_ws_kernel(Args a, int S) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int yp = a.NP + 4, xp = a.xp, stage = a.KP * xp;
  double* ys = reinterpret_cast<double*>(smem_raw);
  double* xs = ys + a.KP * yp;
  uint64_t* full = reinterpret_cast<uint64_t*>(xs + S * stage);
  uint64_t* empty = full + S;
  IDX* xks = reinterpret_cast<IDX*>(empty + S);
  IDX* ccs = xks + a.KP;
  const IDX* xr = static_cast<const IDX*>(a.xr);
  const IDX* xk = static_cast<const IDX*>(a.xk);
  const IDX* yk = static_cast<const IDX*>(a.yk);
  const IDX* yc = static_cast<const IDX*>(a.yc);
  const IDX* cr = static_cast<const IDX*>(a.cr);
  const int nt = 32 * (kWsProd + 8 * CG);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int k = tid; k < a.KP; k += nt) xks[k] = k < a.K ? xk[k] : 0;
  for (int n = tid; n < a.NP; n += nt) ccs[n] = n < a.NC ? static_cast<const IDX*>(a.cc)[n] : 0;
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], kWsProd * 32);   // one cp.async completion arrival per producer thread
      mbar_init(&empty[q], 8);             // one arrival per consumer warp of the group
    }
  }
  for (int e = tid; e < a.KP * a.NP; e += nt) {   // Y, once (zero outside K x NC)
    const int k = e / a.NP, n = e - k * a.NP;
    const bool in = k < a.K && n < a.NC;
    cp_async8(ys + k * yp + n, a.Y + (in ? yk[k] + yc[n] : 0), in);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  const int nblk = (a.R + kRows - 1) / kRows;
  // The CTA's blocks: blockIdx.x, + gridDim.x, ... (the CTAs running together stream one
  // moving window of X and C), or a consecutive range per CTA (TC_SKINNY_CONSEC build flag,
  // measurement: 0.85-0.95x on the HBM-bound strings, though it helps the rank-k kernel's
  // write-only stream; profiles/r02/ab_skinny_walk.txt)
#ifndef TC_SKINNY_CONSEC
  auto blk_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };
  const int nloc = (int)blockIdx.x < nblk ? (nblk - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
#else
  const int per = (nblk + (int)gridDim.x - 1) / (int)gridDim.x;
  auto blk_of = [&](int i) { return (int)blockIdx.x * per + i; };
  const int nloc = max(0, min(per, nblk - (int)blockIdx.x * per));
#endif
  if (warp < kWsProd) {
    // ---- producers: rows-unit lanes take rows 32 h + lane (sub-divided as in the synchronous
    // kernel) for K rows warp, warp + 4, ..; K-unit lanes take 8 consecutive K entries of rows
    // (lane >> 3) + 4 warp + 16 h.
    constexpr int H = ROWS_UNIT ? 2 : 4;
    const int bb = a.bu * a.bv;
    int rl[H], pl[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      if constexpr (ROWS_UNIT) {
        const int e = 32 * h + lane;
        rl[h] = (e % a.bu) * a.bv + (e / a.bu) % a.bv + (e / bb) * bb;
      } else {
        rl[h] = (lane >> 3) + 4 * warp + 16 * h;
      }
      pl[h] = rl[h] + a.sw * (rl[h] >> 4);
    }
    // the row offsets of a block are fetched kWsAhead blocks before its copies are issued
    // (a register ring; the loop is unrolled by kWsAhead so the ring is statically indexed):
    // the producer's own iteration is short, a one-block lookahead would expose the table's
    // load latency on every block
    IDX ro[kWsAhead][H];
    bool rv[kWsAhead][H];
    auto rows = [&](int blk, IDX (&o)[H], bool (&v)[H]) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int r = blk * kRows + rl[h];
        v[h] = blk < nblk && r < a.R;
        o[h] = v[h] ? xr[r] : 0;
      }
    };
#pragma unroll
    for (int d = 0; d < kWsAhead; ++d) rows(d < nloc ? blk_of(d) : nblk, ro[d], rv[d]);
    for (int i0 = 0; i0 < nloc; i0 += kWsAhead) {
#pragma unroll
      for (int d = 0; d < kWsAhead; ++d) {
        const int i = i0 + d;
        if (i >= nloc) break;
        const int q = i % S;
        if (i >= S) mbar_wait(&empty[q], ((i / S) - 1) & 1);
        double* dst = xs + q * stage;
        if (a.dbg & 2) {
        } else if constexpr (ROWS_UNIT) {
#pragma unroll 2
          for (int k = warp; k < a.KP; k += kWsProd) {
            const bool kin = k < a.K;
            const IDX ko = xks[k];
#pragma unroll
            for (int h = 0; h < H; ++h)
              cp_async8_x(dst + k * xp + pl[h], a.X + (ro[d][h] + ko), kin && rv[d][h]);
          }
        } else {
          const int kk = lane & 7;
          for (int k0 = 0; k0 < a.KP; k0 += 8) {
            const int k = k0 + kk;
            if (k < a.KP) {
              const IDX ko = xks[k];
#pragma unroll
              for (int h = 0; h < H; ++h)
                cp_async8_x(dst + k * xp + pl[h], a.X + (ro[d][h] + ko), rv[d][h] && k < a.K);
            }
          }
        }
        mbar_cp_async_arrive(&full[q]);
        rows(i + kWsAhead < nloc ? blk_of(i + kWsAhead) : nblk, ro[d], rv[d]);
      }
    }
    cp_async_wait_all();
    return;
  }
  // ---- consumers: group grp takes the CTA's blocks i = grp, grp + CG, ..; warp cw of the group
  // owns rows wr .. wr + 15 and columns wc .. wc + NP / 2 - 1 of each block
  const int cw = (warp - kWsProd) & 7, grp = (warp - kWsProd) >> 3;
  const int g = lane >> 2, t = lane & 3;
  const int wr = 16 * (cw & 3), wc = (cw >> 2) * (a.NP / 2);
  const int wp = wr + a.sw * (wr >> 4) + g;   // ring position of row wr + g
  double yr[YREG ? kWsMaxK4 : 1][NW];
  if constexpr (YREG) {
#pragma unroll
    for (int k4 = 0; k4 < kWsMaxK4; ++k4)
#pragma unroll
      for (int j = 0; j < NW; ++j)
        yr[k4][j] = 4 * k4 < a.KP ? ys[(4 * k4 + t) * yp + wc + 8 * j + g] : 0.0;
  }
  IDX cco[NW][2];
#pragma unroll
  for (int j = 0; j < NW; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) cco[j][e] = ccs[wc + 8 * j + 2 * t + e];
  const bool full_cols = a.NC == a.NP;
  // C's row offsets: fetched two of the group's blocks ahead (ring indexed by the unrolled d)
  IDX cro[2][2];
  auto crows = [&](int blk, IDX (&o)[2]) {
    const int r0 = blk * kRows + wr + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) o[h] = (blk < nblk && r0 + 8 * h < a.R) ? cr[r0 + 8 * h] : 0;
  };
  crows(grp < nloc ? blk_of(grp) : nblk, cro[0]);
  crows(grp + CG < nloc ? blk_of(grp + CG) : nblk, cro[1]);
  for (int i0 = grp; i0 < nloc; i0 += 2 * CG) {
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const int i = i0 + d * CG;
    if (i >= nloc) break;
    const int blk = blk_of(i);
    const int q = i % S;
    mbar_wait(&full[q], (i / S) & 1);
    const double* xb = xs + q * stage;
    double acc[NW][4];
    if constexpr (YREG) {
#pragma unroll
      for (int j = 0; j < NW; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < kWsMaxK4; ++k4) {
        if (4 * k4 < a.KP && !(a.dbg & 1)) {
          const double a0 = xb[(4 * k4 + t) * xp + wp], a1 = xb[(4 * k4 + t) * xp + wp + 8];
#pragma unroll
          for (int j = 0; j < NW; ++j)
            dmma16x8x4(acc[j][0], acc[j][1], acc[j][2], acc[j][3], a0, a1, yr[k4][j]);
        }
      }
    } else {
      block_mma<IDX, NW>(xb, xp, ys, yp, a.KP, wp - g, wc, g, t, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q]);
    // epilogue from registers: rows wr + g (+8), columns wc + 8 j + 2 t (+1). The streaming
    // stores skip L1 allocation (stores-only f2_00 66.1 -> 56.6 us, whole kernel 123.6 -> 120.8;
    // .cs / an L2 evict-first policy 122.6 / 126.0 us, profiles/r02/ab_skinny_ws.txt)
    const int r0 = blk * kRows + wr + g;
    if (a.dbg & 4) {
    } else if (a.beta == 0.0 && r0 + 8 < a.R && full_cols) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < NW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) st_na(a.C + (cro[d][h] + cco[j][e]), a.alpha * acc[j][2 * h + e]);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (r0 + 8 * h >= a.R) continue;
#pragma unroll
        for (int j = 0; j < NW; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (wc + 8 * j + 2 * t + e >= a.NC) continue;
            double* p = a.C + (cro[d][h] + cco[j][e]);
            double v = a.alpha * acc[j][2 * h + e];
            if (a.beta != 0.0) v = fma(a.beta, *p, v);
            *p = v;
          }
      }
    }
    crows(i + 2 * CG < nloc ? blk_of(i + 2 * CG) : nblk, cro[d]);
  }
  }
}

template <typename IDX, bool ROWS_UNIT, int NW, int CG, bool YREG = true>
static int launch_ws(const Args& a, int nsm, cudaStream_t s, int stages_env) {
  const int fixed = a.KP * (a.NP + 4) * (int)sizeof(double) + (a.KP + a.NP) * (int)sizeof(IDX);
  const int stage = a.KP * a.xp * (int)sizeof(double) + 2 * (int)sizeof(uint64_t);
  // Y in registers (N, K <= 32): 6 stages, 5 blocks (80 KB) in flight per SM; 8 measured
  // slower on f2_00 (130.6 vs 123.4 us), 4 about equal (125.2), 3 139.6 us. Y in shared memory
  // (N, K up to 96, 80): 2 stages -- more in flight measured slower on every such string
  // (f2_02 237.6 / 240.4 / 266.1 us at 2 / 3 / 4 stages; profiles/r02/ab_skinny_ws.txt)
  int S = (227 * 1024 - fixed - 64) / stage;
  const int cap = YREG ? 6 : 2;
  S = S > cap ? cap : S;
  if (stages_env >= 2 && stages_env < S) S = stages_env;
  if (S < 2) return 0;
  const int smem = fixed + S * stage + 64;
  auto kern = tc_skinny_ws_kernel<IDX, ROWS_UNIT, NW, CG, YREG>;
  static std::atomic<int> attr[kMaxDevices];
  if (!ensure_dyn_smem(kern, smem, attr)) return -1;
  const int nblk = (a.R + kRows - 1) / kRows;
  const int grid = nblk < nsm ? nblk : nsm;
  kern<<<grid, 32 * (kWsProd + 8 * CG), smem, s>>>(a, S);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Warp-specialised form (TC_SKINNY_WS = 0 turns it off, _WS_BIG = 0 for the larger resident
// operands only; _CG = 1 | 2 consumer groups (Y in registers), _STAGES caps the ring;
// measurement overrides, read per call). Returns 0 when it does not apply.
template <typename IDX, bool ROWS_UNIT>
static int launch_ws_dir(const Args& a, int nsm, cudaStream_t s) {
  const char* e = getenv("TC_SKINNY_WS");
  if (e && *e == '0') return 0;
  const char* ecg = getenv("TC_SKINNY_WS_CG");
  const char* est = getenv("TC_SKINNY_WS_STAGES");
  const int cg = ecg && *ecg == '1' ? 1 : 2;
  const int st = est ? atoi(est) : 0;
  if (a.NP > 32 || a.KP > 4 * kWsMaxK4) {
    // larger resident operand: Y's fragments from shared memory, one consumer group
    const char* eb = getenv("TC_SKINNY_WS_BIG");
    if (eb && *eb == '0') return 0;
    switch (a.NP / 16) {
      case 1: return launch_ws<IDX, ROWS_UNIT, 1, 1, false>(a, nsm, s, st);
      case 2: return launch_ws<IDX, ROWS_UNIT, 2, 1, false>(a, nsm, s, st);
      case 3: return launch_ws<IDX, ROWS_UNIT, 3, 1, false>(a, nsm, s, st);
      case 4: return launch_ws<IDX, ROWS_UNIT, 4, 1, false>(a, nsm, s, st);
      case 5: return launch_ws<IDX, ROWS_UNIT, 5, 1, false>(a, nsm, s, st);
      default: return launch_ws<IDX, ROWS_UNIT, 6, 1, false>(a, nsm, s, st);
    }
  }
  if (a.NP == 16)
    return cg == 1 ? launch_ws<IDX, ROWS_UNIT, 1, 1>(a, nsm, s, st)
                   : launch_ws<IDX, ROWS_UNIT, 1, 2>(a, nsm, s, st);
  return cg == 1 ? launch_ws<IDX, ROWS_UNIT, 2, 1>(a, nsm, s, st)
                 : launch_ws<IDX, ROWS_UNIT, 2, 2>(a, nsm, s, st);
}

template <typename IDX, bool ROWS_UNIT>
static int launch_dir(const Args& a, int nsm, cudaStream_t s) {
  const int w = launch_ws_dir<IDX, ROWS_UNIT>(a, nsm, s);
  if (w != 0) return w;
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
  // Ring layout. A half-warp's 8-byte cp.async writes land in one shared-memory wavefront only
  // if its 16 rows sit at distinct positions mod 16; the sub-divided row order puts lanes
  // bv rows apart (bu = bv = 8: rows 0, 8, .., 56 -- 4-way conflicts, 13.5 M write wavefronts
  // for 2.1 M of data on f2_00, profiles/r02/ncu/f2_00.summary.txt). Block row r is stored at
  // r + sw (r / 16), sw the smallest skew that minimises the conflicts (the fragment reads
  // take 16 consecutive rows, unaffected by a shift).
  const char* sw_e = getenv("TC_SKINNY_SW");   // override, read per call (TC_SKINNY_SW = 0..4)
  const int sw_env = sw_e && *sw_e ? atoi(sw_e) : -1;
  a.sw = 0;
  if (rows_unit) {
    int best = 1 << 30;
    for (int s = 0; s <= 4; ++s) {
      int cost = 0;
      for (int h0 = 0; h0 < kRows; h0 += 16) {   // the half-warps of the loader
        int cnt[16] = {0}, mx = 0;
        for (int e = h0; e < h0 + 16; ++e) {
          const int bb = a.bu * a.bv;
          const int r = (e % a.bu) * a.bv + (e / a.bu) % a.bv + (e / bb) * bb;
          const int c = ++cnt[(r + s * (r >> 4)) & 15];
          mx = c > mx ? c : mx;
        }
        cost += mx;
      }
      if (cost < best) { best = cost; a.sw = s; }
    }
  }
  if (sw_env >= 0 && sw_env <= 4) a.sw = sw_env;
  a.xp = a.sw ? kXPSkew : kXP;
  const char* dbg_e = getenv("TC_SKINNY_DBG");
  a.dbg = dbg_e ? atoi(dbg_e) : 0;
  if (la.idx64)
    return rows_unit ? launch_dir<long long, true>(a, la.num_sms, stream)
                     : launch_dir<long long, false>(a, la.num_sms, stream);
  return rows_unit ? launch_dir<int, true>(a, la.num_sms, stream)
                   : launch_dir<int, false>(a, la.num_sms, stream);
}

}  // namespace tcb
