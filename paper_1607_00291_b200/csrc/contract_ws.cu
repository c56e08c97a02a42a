// Warp-specialised sm_100a contraction kernel (the production path).
//
//   warps 8-11  producers: gather the A and B tiles of each K step from global memory into a
//               STAGES-deep shared-memory ring with cp.async ("packing", PAPER.md P:593-603,
//               P:696-701): one 16-byte copy per vector of V = 16/sizeof(T) entries that the
//               block-scatter vector (block size V) marks contiguous, V scalar
//               gathers otherwise. When the plan finds every vector of an operand contiguous and
//               16-byte aligned (the operand is block-scatter valid at this granularity,
//               P:703-708) the per-element checks are compiled out (VEC template flag). Copies
//               arrive on the stage's `full` mbarrier as they land.
//   warps 0-7   consumers: wait `full`, run the DMMA micro-kernel on 64x32 warp tiles
//               (mma.sync m16n8k4 f64 -> DMMA.8x8x4; fp32 operands are widened to fp64 on the
//               shared-memory load, so fp32 contractions accumulate in fp64 and round once),
//               release the stage on `empty`; after the serial K loop write
//               alpha*acc + beta*C through rscat_C/cscat_C (beta == 0 never reads C).
//
// The operand layouts in shared memory follow the direction each operand is gathered along
// (its unit-stride bundle), padded so that fragment loads are bank-conflict free.
#include <cstdint>
#include <type_traits>

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
constexpr int GROUP_M = 8;

// Row pads (elements). Fragment loads read 8 rows x 4 columns per half-warp (fp64) or per warp
// (fp32); these pads make every load conflict free: [k][m] rows need LD = 4 mod 16 doubles /
// 8 mod 32 floats, [m][k] rows need 4 mod 16 / 4 mod 32 (20 works for both).
template <typename T> struct Pads;
template <> struct Pads<double> { static constexpr int MN = 4, K = 4; };
template <> struct Pads<float> { static constexpr int MN = 8, K = 4; };

template <typename T, bool VM> struct ALay {   // VM: As[k][m] (gathered along M); else As[m][k]
  static constexpr int LD = VM ? BM + Pads<T>::MN : BK + Pads<T>::K;
  static constexpr int STAGE = VM ? BK * LD : BM * LD;
  __device__ static __forceinline__ int at(int m, int k) { return VM ? k * LD + m : m * LD + k; }
};
template <typename T, bool VK> struct BLay {   // VK: Bs[n][k] (gathered along K); else Bs[k][n]
  static constexpr int LD = VK ? BK + Pads<T>::K : BN + Pads<T>::MN;
  static constexpr int STAGE = VK ? BN * LD : BK * LD;
  __device__ static __forceinline__ int at(int k, int n) { return VK ? n * LD + k : k * LD + n; }
};

template <typename T> __device__ __forceinline__ void cp_async_elem(T* d, const T* s, bool p) {
  if constexpr (sizeof(T) == 8) cp_async8(d, s, p); else cp_async4(d, s, p);
}

// ------------------------------------------------------------------------------------------
// Producer side for one operand X (A or B), in one of two gather modes (V = 16/sizeof(T)):
//  FIXED_VECS: vectors run along the tile's own bundle (M for A, N for B): 128/V vectors,
//              fixed for the whole K loop; producer thread p owns vector p % (128/V) and the
//              K rows rg + V*i (rg = p / (128/V), i < 16/V) of every stage.
//  K_VECS:     vectors run along K: 16/V per stage; thread p owns vector p % (16/V) and the
//              tile rows rb + 8V*i (rb = p / (16/V), i < 16/V), whose offsets it keeps.
// A warp's copy instruction covers 128-512 contiguous bytes of the operand either way.
// VEC: every vector is contiguous and 16-byte aligned (plan-time check), so each slot is one
// 16-byte cp.async with zero-fill outside the extents.
// ------------------------------------------------------------------------------------------
template <typename T, typename IDX, bool FIXED_VECS, bool VEC, int LD>
struct Gather {
  static constexpr int V = 16 / sizeof(T);
  static constexpr int NS = 16 / V;        // slots per producer thread per stage
  IDX o[V];                                // FIXED_VECS: offsets of the vector's entries
  uint32_t vm;                             // FIXED_VECS: bit e = entry e valid, bit V = contiguous
  IDX ro[NS];                              // K_VECS: offsets of the thread's tile rows
  uint32_t rv;                             // K_VECS: bit i = row i in range

  __device__ __forceinline__ void init(const IDX* __restrict__ tab,
                                       const uint8_t* __restrict__ flags, int base,
                                       int extent, int p) {
    if constexpr (FIXED_VECS) {
      const int e = base + V * (p % (128 / V));
      vm = 0;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        o[j] = tab[e + j];
        vm |= (e + j < extent ? 1u : 0u) << j;
      }
      if (e + V - 1 < extent && flags[e / V]) vm |= 1u << V;
    } else {
      const int rb = p / (16 / V);
      rv = 0;
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int r = rb + 8 * V * i;
        ro[i] = tab[base + r];
        rv |= (base + r < extent ? 1u : 0u) << i;
      }
    }
  }

  __device__ __forceinline__ void issue(T* sm, const T* __restrict__ g,
                                        const IDX* __restrict__ ktab,
                                        const uint8_t* __restrict__ kflags, int k0, int K,
                                        int p) {
    if constexpr (FIXED_VECS) {
      const int rg = p / (128 / V);
      IDX kv[NS];
#pragma unroll
      for (int i = 0; i < NS; ++i) kv[i] = __ldg(ktab + k0 + rg + V * i);
      T* d0 = sm + V * (p % (128 / V));
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int r = rg + V * i;
        const bool kin = k0 + r < K;
        T* d = d0 + r * LD;
        const T* p0 = g + (o[0] + kv[i]);
        if constexpr (VEC) {
          cp_async16(d, p0, kin && (vm & 1u));
        } else {
          if (((vm >> V) & 1u) && kin && aligned16(p0)) {
            cp_async16(d, p0, true);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
              cp_async_elem(d + j, g + (o[j] + kv[i]), kin && ((vm >> j) & 1u));
          }
        }
      }
    } else {
      const int kq = p % (16 / V);
      const int k = k0 + V * kq;
      T* d0 = sm + V * kq;
      if constexpr (VEC) {
        const IDX c0 = __ldg(ktab + k);
        const bool kin = k < K;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int r = p / (16 / V) + 8 * V * i;
          cp_async16(d0 + r * LD, g + (ro[i] + c0), kin && ((rv >> i) & 1u));
        }
      } else {
        IDX c[V];
#pragma unroll
        for (int j = 0; j < V; ++j) c[j] = __ldg(ktab + k + j);
        const bool kvec = (k + V - 1 < K) && __ldg(kflags + k / V);
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int r = p / (16 / V) + 8 * V * i;
          const bool rin = (rv >> i) & 1u;
          T* d = d0 + r * LD;
          const T* p0 = g + (ro[i] + c[0]);
          if (kvec && rin && aligned16(p0)) {
            cp_async16(d, p0, true);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
              cp_async_elem(d + j, g + (ro[i] + c[j]), rin && (k + j < K));
          }
        }
      }
    }
  }
};

template <typename T, typename IDX, bool A_VM, bool B_VK, bool A_VEC, bool B_VEC>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_dmma_ws_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                  const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                  const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                  const IDX* __restrict__ rC, const IDX* __restrict__ cC,
                  const uint8_t* __restrict__ vA, const uint8_t* __restrict__ vB,
                  int M, int N, int K, int tiles_m, int tiles_n, double alpha, double beta) {
  using AL = ALay<T, A_VM>;
  using BL = BLay<T, B_VK>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);
  T* Bs = As + STAGES * AL::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      smem_raw + ((STAGES * (AL::STAGE + BL::STAGE) * sizeof(T) + 15) / 16) * 16);
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
    Gather<T, IDX, A_VM, A_VEC, AL::LD> ga;
    Gather<T, IDX, !B_VK, B_VEC, BL::LD> gb;
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
    const T* as = As + s * AL::STAGE;
    const T* bs = Bs + s * BL::STAGE;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = static_cast<double>(as[AL::at(wm + 16 * i + g, 4 * kk + t)]);
        a[i][1] = static_cast<double>(as[AL::at(wm + 16 * i + g + 8, 4 * kk + t)]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = static_cast<double>(bs[BL::at(4 * kk + t, wn + 8 * j + g)]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // epilogue: C[rC[m] + cC[n]] = alpha*acc + beta*C (beta == 0: C not read); computed in fp64,
  // rounded once to T
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
          T* q = C + (rc[2 * i + h] + cc[2 * j + e]);
          double v = alpha * acc[i][j][2 * h + e];
          if (beta != 0.0) v = fma(beta, static_cast<double>(*q), v);
          *q = static_cast<T>(v);
        }
    }
}

template <typename T, typename IDX, bool A_VM, bool B_VK, bool A_VEC, bool B_VEC>
int launch(const LaunchArgs& a, cudaStream_t stream) {
  constexpr int smem =
      ((STAGES * (ALay<T, A_VM>::STAGE + BLay<T, B_VK>::STAGE) * (int)sizeof(T) + 15) / 16) * 16 +
      2 * STAGES * (int)sizeof(uint64_t);
  auto kern = tc_dmma_ws_kernel<T, IDX, A_VM, B_VK, A_VEC, B_VEC>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return -1;
    attr_set = true;
  }
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  kern<<<tiles_m * tiles_n, NTHREADS, smem, stream>>>(
      static_cast<const T*>(a.A), static_cast<const T*>(a.B), static_cast<T*>(a.C),
      static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.vA, a.vB, a.M, a.N, a.K,
      tiles_m, tiles_n, a.alpha, a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename T, typename IDX, bool A_VEC, bool B_VEC>
int dispatch_dir(const LaunchArgs& a, cudaStream_t s) {
  if (a.a_vec_m)
    return a.b_vec_k ? launch<T, IDX, true, true, A_VEC, B_VEC>(a, s)
                     : launch<T, IDX, true, false, A_VEC, B_VEC>(a, s);
  return a.b_vec_k ? launch<T, IDX, false, true, A_VEC, B_VEC>(a, s)
                   : launch<T, IDX, false, false, A_VEC, B_VEC>(a, s);
}

template <typename T>
int dispatch_type(const LaunchArgs& a, cudaStream_t stream) {
  if (a.idx64) return dispatch_dir<T, long long, false, false>(a, stream);
  if (a.a_vec_all)
    return a.b_vec_all ? dispatch_dir<T, int, true, true>(a, stream)
                       : dispatch_dir<T, int, true, false>(a, stream);
  return a.b_vec_all ? dispatch_dir<T, int, false, true>(a, stream)
                     : dispatch_dir<T, int, false, false>(a, stream);
}

}  // namespace ws

int launch_ws(const LaunchArgs& a, cudaStream_t stream) {
  return a.f32 ? ws::dispatch_type<float>(a, stream) : ws::dispatch_type<double>(a, stream);
}

}  // namespace tcb
