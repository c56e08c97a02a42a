// Warp-specialised sm_100a contraction kernel (the production fp64 path).
//
//   warps 8-11  producers: gather the A and B tiles of each K step from global memory into a
//               STAGES-deep shared-memory ring with cp.async ("packing", PAPER.md P:593-603,
//               P:696-701): one 16-byte copy per pair of entries that the block-scatter vector
//               (block size 2) marks contiguous, two 8-byte gathers otherwise. When
//               the plan finds every pair of an operand contiguous and 16-byte aligned (the whole
//               operand is "block-scatter valid" at this granularity) the per-element
//               checks are compiled out (VEC template flag). Copies arrive on the stage's `full`
//               mbarrier as they land (cp.async.mbarrier.arrive.noinc).
//   warps 0-7   consumers: wait `full`, run the DMMA micro-kernel on 64x32 warp tiles
//               (mma.sync m16n8k4 f64 -> DMMA.8x8x4), release the stage on `empty`; after the
//               serial K loop write alpha*acc + beta*C through rscat_C/cscat_C
//               (beta == 0 never reads C).
//
// The operand layouts in shared memory follow the direction each operand is gathered along
// (its unit-stride bundle), padded by 4 doubles so that fragment loads are bank-conflict free.
#include <cstdint>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"

namespace tcb {
namespace ws {

using namespace dev;

constexpr int BM = kBM, BN = kBN, BK = kBK;
constexpr int NCW = 8;                      // consumer warps: 2 (M) x 4 (N), warp tile 64 x 32
constexpr int NPW = 4;                      // producer warps
constexpr int NPT = NPW * 32;               // producer threads
constexpr int NTHREADS = (NCW + NPW) * 32;
constexpr int WM = 64, WN = 32;
constexpr int STAGES = 4;
constexpr int PAD = 4;
constexpr int GROUP_M = 8;

template <bool VM> struct ALay {            // VM: As[k][m] (gathered along M); else As[m][k]
  static constexpr int STAGE = VM ? BK * (BM + PAD) : BM * (BK + PAD);
  static constexpr int LD = VM ? BM + PAD : BK + PAD;
  __device__ static __forceinline__ int at(int m, int k) {
    return VM ? k * (BM + PAD) + m : m * (BK + PAD) + k;
  }
};
template <bool VK> struct BLay {            // VK: Bs[n][k] (gathered along K); else Bs[k][n]
  static constexpr int STAGE = VK ? BN * (BK + PAD) : BK * (BN + PAD);
  static constexpr int LD = VK ? BK + PAD : BN + PAD;
  __device__ static __forceinline__ int at(int k, int n) {
    return VK ? n * (BK + PAD) + k : k * (BN + PAD) + n;
  }
};

// ------------------------------------------------------------------------------------------
// Producer side for one operand X (A or B), in one of two gather modes:
//  FIXED_PAIRS: pairs run along the tile's own bundle (M for A, N for B): 64 pairs, fixed for
//               the whole K loop; producer thread p owns pair p&63 and K rows (p>>6) + 2i.
//  K_PAIRS:     pairs run along K: 8 pairs per stage; thread p owns pair p&7 and tile rows
//               (p>>3) + 16i, whose offsets it keeps in registers.
// Either way a warp's copy instruction covers contiguous 128-512 byte runs of the operand.
// VEC: every pair is contiguous and 16-byte aligned (plan-time block-scatter check), so each
// slot is exactly one 16-byte cp.async with zero-fill outside the extents.
// ------------------------------------------------------------------------------------------
template <typename IDX, bool FIXED_PAIRS, bool VEC, int LD>
struct Gather {
  IDX o0, o1;              // FIXED_PAIRS: offsets of the pair
  uint32_t pm;             // FIXED_PAIRS: bit0 entry0 valid, bit1 entry1 valid, bit2 contiguous
  IDX ro[8];               // K_PAIRS: offsets of the 8 rows
  uint32_t rv;             // K_PAIRS: bit i = row i in range

  __device__ __forceinline__ void init(const IDX* __restrict__ tab,
                                       const uint8_t* __restrict__ flags, int base,
                                       int extent, int p) {
    if constexpr (FIXED_PAIRS) {
      const int e = base + 2 * (p & 63);
      o0 = tab[e];
      o1 = tab[e + 1];
      pm = (e < extent ? 1u : 0u) | (e + 1 < extent ? 2u : 0u) |
           ((e + 1 < extent && flags[e >> 1]) ? 4u : 0u);
    } else {
      rv = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (p >> 3) + 16 * i;
        ro[i] = tab[base + r];
        rv |= (base + r < extent ? 1u : 0u) << i;
      }
    }
  }

  __device__ __forceinline__ void issue(double* sm, const double* __restrict__ g,
                                        const IDX* __restrict__ ktab,
                                        const uint8_t* __restrict__ kflags, int k0, int K,
                                        int p) {
    if constexpr (FIXED_PAIRS) {
      const int rg = p >> 6;
      IDX kv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) kv[i] = __ldg(ktab + k0 + rg + 2 * i);
      double* d0 = sm + 2 * (p & 63);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rg + 2 * i;
        const bool kin = k0 + r < K;
        double* d = d0 + r * LD;
        const double* p0 = g + (o0 + kv[i]);
        if constexpr (VEC) {
          cp_async16(d, p0, kin && (pm & 1u));
        } else {
          if ((pm & 4u) && kin && aligned16(p0)) {
            cp_async16(d, p0, true);
          } else {
            cp_async8(d, p0, kin && (pm & 1u));
            cp_async8(d + 1, g + (o1 + kv[i]), kin && (pm & 2u));
          }
        }
      }
    } else {
      const int kp = p & 7;
      const int k = k0 + 2 * kp;
      const IDX c0 = __ldg(ktab + k);
      const bool kin0 = k < K;
      double* d0 = sm + 2 * kp;
      if constexpr (VEC) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = (p >> 3) + 16 * i;
          cp_async16(d0 + r * LD, g + (ro[i] + c0), kin0 && ((rv >> i) & 1u));
        }
      } else {
        const IDX c1 = __ldg(ktab + k + 1);
        const bool kin1 = k + 1 < K;
        const bool kvec = kin1 && __ldg(kflags + (k >> 1));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = (p >> 3) + 16 * i;
          const bool rin = (rv >> i) & 1u;
          double* d = d0 + r * LD;
          const double* p0 = g + (ro[i] + c0);
          if (kvec && rin && aligned16(p0)) {
            cp_async16(d, p0, true);
          } else {
            cp_async8(d, p0, rin && kin0);
            cp_async8(d + 1, g + (ro[i] + c1), rin && kin1);
          }
        }
      }
    }
  }
};

template <typename IDX, bool A_VM, bool B_VK, bool A_VEC, bool B_VEC>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_dmma_ws_kernel(const double* __restrict__ A, const double* __restrict__ B,
                  double* __restrict__ C,
                  const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                  const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                  const IDX* __restrict__ rC, const IDX* __restrict__ cC,
                  const uint8_t* __restrict__ vA, const uint8_t* __restrict__ vB,
                  int M, int N, int K, int tiles_m, int tiles_n, double alpha, double beta) {
  using AL = ALay<A_VM>;
  using BL = BLay<B_VK>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + STAGES * AL::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * BL::STAGE);
  uint64_t* empty = full + STAGES;

  int tm, tn;
  tile_coords<GROUP_M>(blockIdx.x, tiles_m, tiles_n, &tm, &tn);
  const int m0 = tm * BM, n0 = tn * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], NPT);     // one cp.async arrival per producer thread
      mbar_init(&empty[s], NCW);    // one arrival per consumer warp
    }
  }
  __syncthreads();

  if (warp >= NCW) {
    // ------------------------------- producers -------------------------------
    const int p = threadIdx.x - NCW * 32;
    Gather<IDX, A_VM, A_VEC, AL::LD> ga;
    Gather<IDX, !B_VK, B_VEC, BL::LD> gb;
    // A's tile bundle is M (rA), B's is N (cB); their K tables are cA and rB.
    ga.init(rA, vA, m0, M, p);
    gb.init(cB, vB, n0, N, p);
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      ga.issue(As + s * AL::STAGE, A, cA, vA, kt * BK, K, p);
      gb.issue(Bs + s * BL::STAGE, B, rB, vB, kt * BK, K, p);
      mbar_cp_async_arrive(&full[s]);
    }
    cp_async_wait_all();
    return;
  }

  // --------------------------------- consumers ---------------------------------
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * WM, wn = (warp >> 1) * WN;
  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const double* as = As + s * AL::STAGE;
    const double* bs = Bs + s * BL::STAGE;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = as[AL::at(wm + 16 * i + g, 4 * kk + t)];
        a[i][1] = as[AL::at(wm + 16 * i + g + 8, 4 * kk + t)];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[BL::at(4 * kk + t, wn + 8 * j + g)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: C[rC[m] + cC[n]] = alpha*acc + beta*C (beta == 0: C not read)
  IDX rc[8], cc[8];
  int mm[8], nn[8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = m0 + wm + 16 * i + g + 8 * h;
      mm[2 * i + h] = m;
      rc[2 * i + h] = rC[m];
    }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = n0 + wn + 8 * j + 2 * t + e;
      nn[2 * j + e] = n;
      cc[2 * j + e] = cC[n];
    }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (mm[2 * i + h] >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (nn[2 * j + e] >= N) continue;
          double* q = C + (rc[2 * i + h] + cc[2 * j + e]);
          double v = alpha * acc[i][j][2 * h + e];
          if (beta != 0.0) v = fma(beta, *q, v);
          *q = v;
        }
    }
}

template <typename IDX, bool A_VM, bool B_VK, bool A_VEC, bool B_VEC>
int launch(const LaunchArgs& a, cudaStream_t stream) {
  constexpr int smem = STAGES * (ALay<A_VM>::STAGE + BLay<B_VK>::STAGE) * (int)sizeof(double) +
                       2 * STAGES * (int)sizeof(uint64_t);
  auto kern = tc_dmma_ws_kernel<IDX, A_VM, B_VK, A_VEC, B_VEC>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return -1;
    attr_set = true;
  }
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  kern<<<tiles_m * tiles_n, NTHREADS, smem, stream>>>(
      static_cast<const double*>(a.A), static_cast<const double*>(a.B),
      static_cast<double*>(a.C), static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.vA, a.vB, a.M, a.N, a.K,
      tiles_m, tiles_n, a.alpha, a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename IDX, bool A_VEC, bool B_VEC>
int dispatch_dir(const LaunchArgs& a, cudaStream_t s) {
  if (a.a_vec_m)
    return a.b_vec_k ? launch<IDX, true, true, A_VEC, B_VEC>(a, s)
                     : launch<IDX, true, false, A_VEC, B_VEC>(a, s);
  return a.b_vec_k ? launch<IDX, false, true, A_VEC, B_VEC>(a, s)
                   : launch<IDX, false, false, A_VEC, B_VEC>(a, s);
}

}  // namespace ws

int launch_ws_f64(const LaunchArgs& a, cudaStream_t stream) {
  using namespace ws;
  if (a.idx64) return dispatch_dir<long long, false, false>(a, stream);
  if (a.a_vec_all)
    return a.b_vec_all ? dispatch_dir<int, true, true>(a, stream)
                       : dispatch_dir<int, true, false>(a, stream);
  return a.b_vec_all ? dispatch_dir<int, false, true>(a, stream)
                     : dispatch_dir<int, false, false>(a, stream);
}

}  // namespace tcb
