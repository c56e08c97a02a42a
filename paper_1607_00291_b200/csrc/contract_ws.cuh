#pragma once
// Warp-specialised sm_100a contraction kernel (templates; instantiated by ws_*.cu) (the production path).
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
#include <cstdlib>
#include <type_traits>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"
#include "sched.cuh"

namespace tcb {
namespace ws {

using namespace dev;
using namespace sched;

constexpr int BM = kBM, BN = kBN, BK = kBK;
constexpr int NCW = 8;                      // consumer warps: 2 (M) x 4 (N), warp tile 64 x 32
constexpr int NPW = 4;                      // producer warps
constexpr int NPT = NPW * 32;               // producer threads
constexpr int NTHREADS = (NCW + NPW) * 32;
constexpr int WM = 64, WN = 32;
constexpr int kWarpTab = WM + WN;           // C scatter entries per consumer warp and tile
// Ring depth per element type. fp32 keeps 4 stages although its K step is twice as short: the
// element gathers (cp.async 4 B, cached in L1) need the L1 share that a deeper ring plus the
// epilogue staging buffers would take from the 256 KB L1/shared array (measured: 8 stages cost
// up to 13% on cfg4 fp32 cases with element-gathered operands, profiles/r01/ab_stages_f32.txt).
#ifndef TC_STAGES_F32
#define TC_STAGES_F32 4
#endif
#ifndef TC_STAGES_F64
#define TC_STAGES_F64 4
#endif
template <typename T> constexpr int stages() {
  return sizeof(T) == 4 ? TC_STAGES_F32 : TC_STAGES_F64;
}
// FFMA epilogue staging (fp32): per consumer warp its 64 x 32 accumulator block as [n][m]
// floats, row pitch kEpiLD (a multiple of 4 for 16-byte accesses)
constexpr int kEpiLD = 64 + 4;
constexpr int kEpiWarpFloats = 32 * kEpiLD;
// DMMA epilogue staging (fp64, when C's unit stride runs along M): per consumer warp 16 rows
// x 32 columns of its block at a time, [n][m] doubles with pitch kEpiDLD; four passes. Off by
// default: measured slower than the direct fragment stores (which already fill whole sectors)
// on the small-K families (f1 k16: 0.85 -> 0.72 of DGEMM; profiles/r01/ab_dmma_staged.txt).
#ifndef TC_DMMA_STAGED
#define TC_DMMA_STAGED 0
#endif
constexpr int kEpiDLD = 16 + 4;
// Edge tiles multiply only the m16 / n8 blocks of each warp tile that hold data (stage_edge);
// TC_DMMA_EDGE=0 builds the variant without (measurement A/B).
#ifndef TC_DMMA_EDGE
#define TC_DMMA_EDGE 1
#endif
constexpr int kEpiWarpDoubles = 32 * kEpiDLD;
constexpr int kSmemLimit = 232448;   // 227 KB of dynamic shared memory per CTA
// Tile rasterisation group height. With K in the tens of thousands a CTA's A and B panels are
// tens of MB, and the CTAs of a wave drift apart in K faster than L2 (126 MB, turned over every
// ~80 us at cfg5's miss rate) can bridge, so sharing within a wave is small; what L2 does keep
// is the A panels of the few tile rows that consecutive waves revisit. Two rows per group keep
// those resident: cfg5 DRAM reads 3.82 TB (8 rows) -> 3.02 TB per launch, same time
// (profiles/r01/l2_group_sweep_cfg5.txt); neutral on every other suite case.
#ifndef TC_GROUP_M
#define TC_GROUP_M 2
#endif
constexpr int GROUP_M = TC_GROUP_M;
// setmaxnreg budgets: 128 x 56 + 256 x 224 = 64512 <= 65536 registers per SM, and per SMSP
// (warps w, w+4, w+8) 224 + 224 + 56 = 504 <= 512 registers per lane.
constexpr int kProducerRegs = 64;
constexpr int kConsumerRegs = 216;

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
// One vector of 16/sizeof(T) consecutive elements whose start may not be 16-byte aligned (the
// smem destination always is): one 16-byte copy when aligned, else the widest copies whose
// source and destination are both aligned.
template <typename T>
__device__ __forceinline__ void copy_contig(T* d, const T* p) {
  if (aligned16(p)) {
    cp_async16(d, p, true);
  } else if constexpr (sizeof(T) == 4) {
    if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
      cp_async8(d, p, true);
      cp_async8(d + 2, p + 2, true);
    } else {   // source and destination 8-byte alignments differ: element copies
#pragma unroll
      for (int j = 0; j < 4; ++j) cp_async4(d + j, p + j, true);
    }
  } else {
    cp_async8(d, p, true);
    cp_async8(d + 1, p + 1, true);
  }
}

template <typename T, typename IDX, bool FIXED_VECS, bool VEC, int LD>
struct Gather {
  static constexpr int V = 16 / sizeof(T);
  static constexpr int NS = 16 / V;        // slots per producer thread per stage
  IDX o[V];                                // FIXED_VECS: offsets of the vector's entries
  uint32_t vm;                             // FIXED_VECS: bit e = entry e valid, bit V = contiguous
  IDX ro[NS];                              // K_VECS: offsets of the thread's tile rows
  uint32_t rv;                             // K_VECS: bit i = row i in range
  // K-table entries of the next stage, loaded one stage ahead (load_k) so that their latency
  // overlaps the wait for a free ring slot instead of delaying the copies
  IDX kv[FIXED_VECS ? NS : V];
  bool kvec;                               // K_VECS: the thread's V K-entries are contiguous

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

  // K-table entries this thread needs for the stage starting at k0 (tables are padded by at
  // least 128 entries, so reads past K are in bounds; their copies are predicated off).
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab,
                                         const uint8_t* __restrict__ kflags, int k0, int K,
                                         int p) {
    if constexpr (FIXED_VECS) {
      const int rg = p / (128 / V);
#pragma unroll
      for (int i = 0; i < NS; ++i) kv[i] = __ldg(ktab + k0 + rg + V * i);
    } else {
      const int k = k0 + V * (p % (16 / V));
      if constexpr (VEC) {
        kv[0] = __ldg(ktab + k);
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j) kv[j] = __ldg(ktab + k + j);
        kvec = (k + V - 1 < K) && __ldg(kflags + k / V);
      }
    }
  }

  __device__ __forceinline__ void issue(T* sm, const T* __restrict__ g, int k0, int K, int p) {
    if constexpr (FIXED_VECS) {
      const int rg = p / (128 / V);
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
          if (((vm >> V) & 1u) && kin) {
            copy_contig(d, p0);
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
        const bool kin = k < K;
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int r = p / (16 / V) + 8 * V * i;
          cp_async16(d0 + r * LD, g + (ro[i] + kv[0]), kin && ((rv >> i) & 1u));
        }
      } else {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int r = p / (16 / V) + 8 * V * i;
          const bool rin = (rv >> i) & 1u;
          T* d = d0 + r * LD;
          const T* p0 = g + (ro[i] + kv[0]);
          if (kvec && rin) {
            copy_contig(d, p0);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j)
              cp_async_elem(d + j, g + (ro[i] + kv[j]), rin && (k + j < K));
          }
        }
      }
    }
  }
};

// Coalesced element gather (mode 2), for operands whose 16-byte vectors are often not
// contiguous or not aligned (short or odd unit-stride runs): every copy moves one element, and
// the 32 lanes of a warp take 32 consecutive entries of the gather direction, so when the
// entries are consecutive addresses one warp instruction reads one 128-byte (fp32) or 256-byte
// (fp64) run instead of 32 lane-strided pieces.
//  FIXED_VECS (gathered along the tile's own bundle, [k][row] layout): lane l owns bundle
//              entries l + 32 j (j < 4), fixed for the tile; warp w owns K rows 4 w + i.
//  K_VECS     ([row][k] layout): lane l owns K entry l % 16 of every stage and tile rows
//              32 w + 2 q + l / 16 (q < 16), whose offsets it keeps.
// Each thread issues 16 element copies per stage either way.
template <typename T, typename IDX, bool FIXED_VECS, int LD>
struct GatherElem {
  static constexpr int NR = FIXED_VECS ? 4 : 16;   // fixed offsets per thread
  IDX o[NR];
  uint32_t valid;                                  // bit q: fixed entry q in range
  IDX kv[FIXED_VECS ? 4 : 1];                      // next stage's K entries (load_k)

  __device__ __forceinline__ void init(const IDX* __restrict__ tab, const uint8_t*, int base,
                                       int extent, int p) {
    const int w = p >> 5, l = p & 31;
    valid = 0;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const int e = FIXED_VECS ? base + l + 32 * q : base + 32 * w + 2 * q + (l >> 4);
      o[q] = tab[e];
      valid |= (e < extent ? 1u : 0u) << q;
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, const uint8_t*, int k0,
                                         int, int p) {
    if constexpr (FIXED_VECS) {
#pragma unroll
      for (int i = 0; i < 4; ++i) kv[i] = __ldg(ktab + k0 + 4 * (p >> 5) + i);
    } else {
      kv[0] = __ldg(ktab + k0 + (p & 15));
    }
  }
  __device__ __forceinline__ void issue(T* sm, const T* __restrict__ g, int k0, int K, int p) {
    const int w = p >> 5, l = p & 31;
    if constexpr (FIXED_VECS) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * w + i;
        const bool kin = k0 + r < K;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          cp_async_elem(sm + r * LD + l + 32 * j, g + (o[j] + kv[i]), kin && ((valid >> j) & 1u));
      }
    } else {
      const int kk = l & 15;
      const bool kin = k0 + kk < K;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int r = 32 * w + 2 * q + (l >> 4);
        cp_async_elem(sm + r * LD + kk, g + (o[q] + kv[0]), kin && ((valid >> q) & 1u));
      }
    }
  }
};

// Transposing element gather (mode 3, fp32 A only): A is read along K (its unit stride) but
// written to the [k][m] layout, so that an fp32 contraction whose A and B are both K-contiguous
// runs the PAIR_R micro-kernel (one accumulator set) instead of PAIR_K (two). Lane l of warp w
// takes K entry 8 h + (l & 7) and tile row 32 w + 4 g + (l >> 3) (h < 2, g < 8): each warp
// instruction reads four 32-byte runs and writes 16 distinct banks (2-way conflicts).
template <typename T, typename IDX, int LD>
struct GatherElemT {
  IDX o[8];
  uint32_t valid;
  IDX kv[2];
  __device__ __forceinline__ void init(const IDX* __restrict__ tab, const uint8_t*, int base,
                                       int extent, int p) {
    const int w = p >> 5, l = p & 31;
    valid = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const int e = base + 32 * w + 4 * g + (l >> 3);
      o[g] = tab[e];
      valid |= (e < extent ? 1u : 0u) << g;
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, const uint8_t*, int k0,
                                         int, int p) {
#pragma unroll
    for (int h = 0; h < 2; ++h) kv[h] = __ldg(ktab + k0 + 8 * h + (p & 7));
  }
  __device__ __forceinline__ void issue(T* sm, const T* __restrict__ g, int k0, int K, int p) {
    const int w = p >> 5, l = p & 31;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 8 * h + (l & 7);
      const bool kin = k0 + kk < K;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        cp_async_elem(sm + kk * LD + 32 * w + 4 * q + (l >> 3), g + (o[q] + kv[h]),
                      kin && ((valid >> q) & 1u));
    }
  }
};

// Gather mode per operand: 0 = every vector contiguous and aligned (one 16-byte copy each),
// 1 = per-vector check (16-byte copy where contiguous, element copies elsewhere),
// 2 = coalesced element copies (GatherElem), 3 = transposing element copies (GatherElemT).
template <typename T, typename IDX, bool FIXED_VECS, int MODE, int LD> struct GatherSel {
  using type = Gather<T, IDX, FIXED_VECS, MODE == 0, LD>;
};
template <typename T, typename IDX, bool FIXED_VECS, int LD> struct GatherSel<T, IDX, FIXED_VECS, 2, LD> {
  using type = GatherElem<T, IDX, FIXED_VECS, LD>;
};
template <typename T, typename IDX, bool FIXED_VECS, int LD> struct GatherSel<T, IDX, FIXED_VECS, 3, LD> {
  using type = GatherElemT<T, IDX, LD>;
};

// ------------------------------------------------------------------------------------------
// Micro-kernels (register-tiled C += A.B over one K step). Each thread owns
// an 8 x 8 block of its warp's 64 x 32 tile, exposed as acc[r][c] at (row(r), col(c)), so the
// epilogue is shared.
//  MicroDmma: mma.sync m16n8k4 f64 (DMMA.8x8x4) with fp64 accumulators; fp32 operands are
//             widened on the shared-memory load (fp64 accumulation, one rounding at the end).
//  MicroFfma: fp32 FFMA outer products with fp32 accumulators (the FMA micro-kernel of the
//             north star for fp32): 16-byte shared loads along each layout's contiguous
//             direction, 64 FFMA per 16 loaded values.
// ------------------------------------------------------------------------------------------
// Consumer warp w of the DMMA micro-kernel owns rows dmma_wm(w) .. + 63 and columns
// dmma_wn(w) .. + 31 of the tile. Warps w and w + 4 share a sub-partition (SMSP, one DMMA unit):
// they take opposite row halves and column quarters two apart, so on a ragged edge tile (rows
// or columns cut, the cut-off warps skipping their empty MMAs, stage_edge) every SMSP keeps part
// of the work -- the tile's time per K step is its busiest SMSP's (dmma_tile_weight).
#ifndef TC_DMMA_OLDMAP
__host__ __device__ constexpr int dmma_wm(int w) { return ((w >> 2) & 1) * WM; }
__host__ __device__ constexpr int dmma_wn(int w) { return ((w & 3) ^ (2 * ((w >> 2) & 1))) * WN; }
#else   // measurement A/B: the previous map (warp w: rows (w & 1), columns w >> 1)
__host__ __device__ constexpr int dmma_wm(int w) { return (w & 1) * WM; }
__host__ __device__ constexpr int dmma_wn(int w) { return (w >> 1) * WN; }
#endif

template <typename T, bool A_VM, bool B_VK>
struct MicroDmma {
  using Acc = double;
  using AL = ALay<T, A_VM>;
  using BL = BLay<T, B_VK>;
  Acc acc[8][8];      // row r = 2i+h: m = wm + 16i + g + 8h; col c = 2j+e: n = wn + 8j + 2t + e
  int wm, wn, g, t;
  __device__ __forceinline__ void setup(int warp, int lane) {
    g = lane >> 2; t = lane & 3; wm = dmma_wm(warp); wn = dmma_wn(warp);
  }
  __device__ __forceinline__ int row(int r) const { return wm + 16 * (r >> 1) + g + 8 * (r & 1); }
  __device__ __forceinline__ int col(int c) const { return wn + 8 * (c >> 1) + 2 * t + (c & 1); }
  __device__ __forceinline__ double value(int r, int c) const { return acc[r][c]; }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
  }
  __device__ __forceinline__ void stage(const T* as, const T* bs) {
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = static_cast<double>(as[AL::at(wm + 16 * i + g, 4 * kk + t)]);
        a[i][1] = static_cast<double>(as[AL::at(wm + 16 * i + g + 8, 4 * kk + t)]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        b[j] = static_cast<double>(bs[BL::at(4 * kk + t, wn + 8 * j + g)]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dmma16x8x4(acc[2 * i][2 * j], acc[2 * i][2 * j + 1], acc[2 * i + 1][2 * j],
                     acc[2 * i + 1][2 * j + 1], a[i][0], a[i][1], b[j]);
    }
  }
  // ragged tile edges (and / or the last, partial K step): only the ni m16 blocks and nj n8
  // blocks of the warp tile that hold rows < M and columns < N, and the nk4 groups of 4 k that
  // hold data (warp-uniform bounds). A 128 x 128 tile over a 323-row edge (fig:bench's
  // ab-cad-dcb) then multiplies 336 rows instead of 384.
  __device__ __forceinline__ void stage_edge(const T* as, const T* bs, int nk4, int ni, int nj) {
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      if (kk >= nk4) break;
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = static_cast<double>(as[AL::at(wm + 16 * i + g, 4 * kk + t)]);
        a[i][1] = static_cast<double>(as[AL::at(wm + 16 * i + g + 8, 4 * kk + t)]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        b[j] = static_cast<double>(bs[BL::at(4 * kk + t, wn + 8 * j + g)]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i >= ni) break;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= nj) break;
          dmma16x8x4(acc[2 * i][2 * j], acc[2 * i][2 * j + 1], acc[2 * i + 1][2 * j],
                     acc[2 * i + 1][2 * j + 1], a[i][0], a[i][1], b[j]);
        }
      }
    }
  }
  // last, partial K step: only the nk4 groups of 4 k that hold data (the rest is zero-filled)
  __device__ __forceinline__ void stage_tail(const T* as, const T* bs, int nk4) {
    for (int kk = 0; kk < nk4; ++kk) {
      double a[4][2], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i][0] = static_cast<double>(as[AL::at(wm + 16 * i + g, 4 * kk + t)]);
        a[i][1] = static_cast<double>(as[AL::at(wm + 16 * i + g + 8, 4 * kk + t)]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        b[j] = static_cast<double>(bs[BL::at(4 * kk + t, wn + 8 * j + g)]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          dmma16x8x4(acc[2 * i][2 * j], acc[2 * i][2 * j + 1], acc[2 * i + 1][2 * j],
                     acc[2 * i + 1][2 * j + 1], a[i][0], a[i][1], b[j]);
    }
  }
};

// d0 += a0 * b0, d1 += a1 * b1 as one packed fp32x2 FMA (SASS FFMA2; a0 == a1 becomes the
// scalar-broadcast form). Two FMAs per lane per issue slot.
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1) {
  unsigned long long d, x, y;
  asm("mov.b64 %0, {%1,%2};" : "=l"(d) : "f"(d0), "f"(d1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(y) : "f"(b0), "f"(b1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(x), "l"(y));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}

template <bool A_VM, bool B_VK>
struct MicroFfma {
  using Acc = float;
  using AL = ALay<float, A_VM>;
  using BL = BLay<float, B_VK>;
  // FFMA2 pairs two accumulators whose operands sit in adjacent registers of a 16-byte load:
  //  PAIR_C: (acc[r][c], acc[r][c+1]) with b[k][c..c+1] from one load ([k][n] layout of B)
  //  PAIR_R: (acc[r][c], acc[r+1][c]) with a[k][r..r+1] ([k][m] layout of A, B is [n][k])
  //  PAIR_K: (acc[r][c], acc2[r][c]) = even / odd k partial sums ([m][k] and [n][k] layouts)
  static constexpr int PAIR_C = 0, PAIR_R = 1, PAIR_K = 2;
#ifndef TC_FFMA_PAIRK
#define TC_FFMA_PAIRK 1
#endif
  static constexpr int MODE = !B_VK ? PAIR_C : (A_VM ? PAIR_R : (TC_FFMA_PAIRK ? PAIR_K : PAIR_C));
  Acc acc[8][8];
  Acc acc2[MODE == PAIR_K ? 8 : 1][MODE == PAIR_K ? 8 : 1];
  int wm, wn, tm, tn;     // lane = tm + 8 tn (tm 0..7 over M, tn 0..3 over N)
  __device__ __forceinline__ void setup(int warp, int lane) {
    tm = lane & 7; tn = lane >> 3; wm = (warp & 1) * WM; wn = (warp >> 1) * WN;
  }
  // [k][m] rows: two runs of 4 consecutive m (16-byte loads); [m][k]: rows tm + 8r (a 16-byte
  // load gives 4 consecutive k). Same for columns of B ([k][n] runs / [n][k] rows tn + 4c).
  __device__ __forceinline__ int row(int r) const {
    return A_VM ? wm + (r < 4 ? 4 * tm + r : 32 + 4 * tm + r - 4) : wm + tm + 8 * r;
  }
  __device__ __forceinline__ int col(int c) const {
    return !B_VK ? wn + (c < 4 ? 4 * tn + c : 16 + 4 * tn + c - 4) : wn + tn + 4 * c;
  }
  __device__ __forceinline__ float value(int r, int c) const {
    if constexpr (MODE == PAIR_K) return acc[r][c] + acc2[r][c];
    else return acc[r][c];
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    if constexpr (MODE == PAIR_K) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc2[r][c] = 0.f;
    }
  }
  // fragments of one group of 4 k (PAIR_C / PAIR_R) or 2 k (PAIR_K)
  __device__ __forceinline__ void load4(const float* as, const float* bs, int kk, float (&a)[4][8],
                                        float (&b)[4][8]) const {
    if constexpr (A_VM) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 x = *reinterpret_cast<const float4*>(as + (4 * kk + k) * AL::LD + wm + 4 * tm);
        const float4 y = *reinterpret_cast<const float4*>(as + (4 * kk + k) * AL::LD + wm + 32 + 4 * tm);
        a[k][0] = x.x; a[k][1] = x.y; a[k][2] = x.z; a[k][3] = x.w;
        a[k][4] = y.x; a[k][5] = y.y; a[k][6] = y.z; a[k][7] = y.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float4 x = *reinterpret_cast<const float4*>(as + (wm + tm + 8 * r) * AL::LD + 4 * kk);
        a[0][r] = x.x; a[1][r] = x.y; a[2][r] = x.z; a[3][r] = x.w;
      }
    }
    if constexpr (!B_VK) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 x = *reinterpret_cast<const float4*>(bs + (4 * kk + k) * BL::LD + wn + 4 * tn);
        const float4 y = *reinterpret_cast<const float4*>(bs + (4 * kk + k) * BL::LD + wn + 16 + 4 * tn);
        b[k][0] = x.x; b[k][1] = x.y; b[k][2] = x.z; b[k][3] = x.w;
        b[k][4] = y.x; b[k][5] = y.y; b[k][6] = y.z; b[k][7] = y.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 x = *reinterpret_cast<const float4*>(bs + (wn + tn + 4 * c) * BL::LD + 4 * kk);
        b[0][c] = x.x; b[1][c] = x.y; b[2][c] = x.z; b[3][c] = x.w;
      }
    }
  }
  __device__ __forceinline__ void load2(const float* as, const float* bs, int k2, float (&a)[2][8],
                                        float (&b)[2][8]) const {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float2 x = *reinterpret_cast<const float2*>(as + (wm + tm + 8 * r) * AL::LD + 2 * k2);
      a[0][r] = x.x; a[1][r] = x.y;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float2 x = *reinterpret_cast<const float2*>(bs + (wn + tn + 4 * c) * BL::LD + 2 * k2);
      b[0][c] = x.x; b[1][c] = x.y;
    }
  }
  __device__ __forceinline__ void fma4(const float (&a)[4][8], const float (&b)[4][8]) {
    if constexpr (MODE == PAIR_C) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; c += 2)
            ffma2(acc[r][c], acc[r][c + 1], a[k][r], a[k][r], b[k][c], b[k][c + 1]);
    } else {   // PAIR_R
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int r = 0; r < 8; r += 2)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            ffma2(acc[r][c], acc[r + 1][c], a[k][r], a[k][r + 1], b[k][c], b[k][c]);
    }
  }
  __device__ __forceinline__ void fma2k(const float (&a)[2][8], const float (&b)[2][8]) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        ffma2(acc[r][c], acc2[r][c], a[0][r], a[1][r], b[0][c], b[1][c]);
  }
  // one K step: the fragments of the next k group load while the current one is consumed
  __device__ __forceinline__ void stage(const float* as, const float* bs) {
    if constexpr (MODE == PAIR_K) {
#pragma unroll 2
      for (int k2 = 0; k2 < BK / 2; ++k2) {
        float a[2][8], b[2][8];
        load2(as, bs, k2, a, b);
        fma2k(a, b);
      }
    } else {
      float a[2][4][8], b[2][4][8];
      load4(as, bs, 0, a[0], b[0]);
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        if (kk + 1 < BK / 4) load4(as, bs, kk + 1, a[(kk + 1) & 1], b[(kk + 1) & 1]);
        fma4(a[kk & 1], b[kk & 1]);
      }
    }
  }
};

template <typename T, bool FFMA, bool A_VM, bool B_VK> struct MicroSel {
  using type = MicroDmma<T, A_VM, B_VK>;
};
template <bool A_VM, bool B_VK> struct MicroSel<float, true, A_VM, B_VK> {
  using type = MicroFfma<A_VM, B_VK>;
};

// Stores of C. TC_C_STREAM_STORE=1 sends final values with the streaming hint (st.global.cs,
// evict-first; a stream-K piece that a later piece reads back is stored normally). Off: it
// measured slower, most on the C-write-bound shapes (f1 k16 0.88 -> 0.70, f2 K=18 strings
// 0.84-0.90 -> 0.70-0.73 of DGEMM; profiles/r01/ab_stream_store.txt).
#ifndef TC_C_STREAM_STORE
#define TC_C_STREAM_STORE 0
#endif
template <typename T>
__device__ __forceinline__ void store_c(T* p, T v, bool keep) {
  if (TC_C_STREAM_STORE && !keep) __stcs(p, v);
  else *p = v;
}

// Stream-K accumulation of an fp64 piece: C += v as a reduction at L2 (red.global.add.f64,
// one IEEE add, the same result as the load-add-store it replaces; the fix-up order is still set
// by the per-tile flags, and the piece's fence before publishing waits for the reductions). The
// pieces of a split tile then no longer pay a load round trip per chunk of C between links of
// the fix-up chain. TC_SK_RED=0 builds the load-add-store form (measurement A/B).
#ifndef TC_SK_RED
#define TC_SK_RED 1
#endif
__device__ __forceinline__ void red_add_c(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

// ---- cluster split-K (Sched::csplit) ----------------------------------------------------------
// Each CTA of a cluster leaves its fp64 partial tile in its own (now idle) ring memory as
// part[col][row] (pitch kPP), the cluster synchronises, and CTA r sums rows [r 128 / S,
// (r + 1) 128 / S) of all S partials, read through distributed shared memory in rank order,
// then writes alpha * sum + beta * C. A second cluster barrier keeps every CTA's shared memory
// alive until all reads are done.
constexpr int kPP = BM + 4;   // partial tile pitch (doubles), [col][row]
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ double ld_dsmem(uint32_t local, uint32_t rank) {
  uint32_t remote;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

__device__ __forceinline__ void producers_sync() {
  asm volatile("bar.sync 2, %0;\n" ::"n"(NPT) : "memory");
}
// Bounded wait (about 20 us) for the wave counter: a CTA that is not co-resident with the rest
// of the grid can only delay the others, never deadlock them.
constexpr long long kWaveTimeout = 40000;
__device__ __forceinline__ void wave_wait(const int* ctr, unsigned target) {
  const long long t0 = clock64();
  while ((int)((unsigned)ld_acquire(ctr) - target) < 0) {
    if (clock64() - t0 > kWaveTimeout) break;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void wave_arrive(int* ctr) {
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctr) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory");
}

// Shared memory: the ring, the full/empty barriers, the per-warp C-table slices and (FFMA) the
// per-warp epilogue staging buffers; the ring is as deep as stages<T>() allows within 227 KB.
template <typename T, bool A_VM, bool B_VK, typename IDX, bool FFMA>
constexpr int smem_bytes(int stages_) {
  return ((stages_ * (ALay<T, A_VM>::STAGE + BLay<T, B_VK>::STAGE) * (int)sizeof(T) + 15) / 16) * 16 +
         2 * stages_ * (int)sizeof(uint64_t) + NCW * kWarpTab * (int)sizeof(IDX) +
         (FFMA ? NCW * kEpiWarpFloats * (int)sizeof(float)
               : (TC_DMMA_STAGED ? NCW * kEpiWarpDoubles * (int)sizeof(double) : 0));
}
template <typename T, bool A_VM, bool B_VK, typename IDX, bool FFMA>
constexpr int ring_stages() {
  int st = stages<T>();
  while (st > 2 && smem_bytes<T, A_VM, B_VK, IDX, FFMA>(st) > kSmemLimit) --st;
  return st;
}

// cluster split-K needs fp64 DMMA and a ring at least as large as the partial tile
template <typename T, bool A_VM, bool B_VK, typename IDX, bool FFMA>
constexpr bool csk_fits() {
  return !FFMA && std::is_same<T, double>::value &&
         ring_stages<T, A_VM, B_VK, IDX, FFMA>() * (ALay<T, A_VM>::STAGE + BLay<T, B_VK>::STAGE) *
                 (int)sizeof(T) >= BN * kPP * (int)sizeof(double);
}

template <typename T, typename IDX, bool A_VM, bool B_VK, int A_MODE, int B_MODE, bool FFMA>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_dmma_ws_kernel(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                  const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                  const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                  const IDX* __restrict__ rC, const IDX* __restrict__ cC,
                  const uint8_t* __restrict__ vA, const uint8_t* __restrict__ vB,
                  int M, int N, int K, int tiles_m, int tiles_n, double alpha, double beta,
                  Sched sched, int* __restrict__ flags, bool c_lanes_n) {
  using AL = ALay<T, A_VM>;
  using BL = BLay<T, B_VK>;
  constexpr int STAGES = ring_stages<T, A_VM, B_VK, IDX, FFMA>();
  constexpr bool kCsk = csk_fits<T, A_VM, B_VK, IDX, FFMA>();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);
  T* Bs = As + STAGES * AL::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      smem_raw + ((STAGES * (AL::STAGE + BL::STAGE) * sizeof(T) + 15) / 16) * 16);
  uint64_t* empty = full + STAGES;
  // per consumer warp: the C scatter entries of its 64 rows and 32 columns of the current tile
  IDX* wtab = reinterpret_cast<IDX*>(empty + STAGES) + (threadIdx.x >> 5) * kWarpTab;
  float* epi = reinterpret_cast<float*>(reinterpret_cast<IDX*>(empty + STAGES) + NCW * kWarpTab) +
               (threadIdx.x >> 5) * kEpiWarpFloats;
  double* epid = reinterpret_cast<double*>(reinterpret_cast<IDX*>(empty + STAGES) + NCW * kWarpTab) +
                 (threadIdx.x >> 5) * kEpiWarpDoubles;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], NPT);     // one cp.async arrival per producer thread
      mbar_init(&empty[s], NCW);    // one arrival per consumer warp
    }
  }
  __syncthreads();

  WorkIter wi;
  wi.init(sched, blockIdx.x);
  int tile, kb, ke;
  bool sk;
  uint32_t it = 0;   // global K-iteration counter of this CTA: ring stage and phase

  if (warp >= NCW) {
    // ------------------------------- producers -------------------------------
    // registers move from the producer warpgroup to the two consumer warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    const int p = threadIdx.x - NCW * 32;
    typename GatherSel<T, IDX, A_VM, A_MODE, AL::LD>::type ga;
    typename GatherSel<T, IDX, !B_VK, B_MODE, BL::LD>::type gb;
    int* wave_ctr = flags + 2 * sched.P;   // after the stream-K flags
    int dp_items = 0;
    while (wi.next(tile, kb, ke, sk)) {
      if (!sk && sched.wave_sync && dp_items > 0) {
        if (p == 0) wave_wait(wave_ctr, sched.wave_base + (unsigned)(dp_items * sched.P));
        producers_sync();
      }
      int tm, tn;
      tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
      // A's tile bundle is M (rA), B's is N (cB); their K tables are cA and rB.
      ga.init(rA, vA, tm * BM, M, p);
      gb.init(cB, vB, tn * BN, N, p);
      ga.load_k(cA, vA, kb * BK, K, p);
      gb.load_k(rB, vB, kb * BK, K, p);
      for (int kt = kb; kt < ke; ++kt, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        ga.issue(As + s * AL::STAGE, A, kt * BK, K, p);
        gb.issue(Bs + s * BL::STAGE, B, kt * BK, K, p);
        mbar_cp_async_arrive(&full[s]);
        ga.load_k(cA, vA, (kt + 1) * BK, K, p);   // next stage's K entries (padded tables)
        gb.load_k(rB, vB, (kt + 1) * BK, K, p);
      }
      if (!sk && sched.wave_sync) {
        if (p == 0) wave_arrive(wave_ctr);
        ++dp_items;
      }
    }
    cp_async_wait_all();
    if (sched.csplit) {   // the consumers' two cluster barriers (partials written, sums read)
      cluster_sync_all();
      cluster_sync_all();
    }
    return;
  }

  // --------------------------------- consumers ---------------------------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
  typename MicroSel<T, FFMA, A_VM, B_VK>::type mk;
  mk.setup(warp, lane);
  while (wi.next(tile, kb, ke, sk)) {
    int tm, tn;
    tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
    const int m0 = tm * BM, n0 = tn * BN;
    // fetch this warp's rC / cC entries for the epilogue now (cp.async into its private smem;
    // tables are padded past M, N), so their latency hides behind the K loop
    for (int q = lane; q < kWarpTab; q += 32) {
      const IDX* src = q < WM ? rC + (m0 + mk.wm + q) : cC + (n0 + mk.wn + q - WM);
      if constexpr (sizeof(IDX) == 8) cp_async8(wtab + q, src, true);
      else cp_async4(wtab + q, src, true);
    }
    if (beta != 0.0 && kb == 0 && ke - kb >= 4) {
      // pull the warp's 64 x 32 block of C into L2 while the K loop runs: lane l takes column
      // l and four 16-row runs (one 128-byte line each when C is contiguous along M)
      const int n = n0 + mk.wn + lane;
      if (n < N) {
        const IDX c = cC[n];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int m = m0 + mk.wm + 16 * q;
          if (m < M) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(C + (rC[m] + c)));
        }
      }
    }
    mk.zero();
    // m16 / n8 blocks of this warp's 64 x 32 tile that hold rows < M, columns < N
    int edge_mi = 4, edge_nj = 4;
    if constexpr (!FFMA && TC_DMMA_EDGE) {
      edge_mi = (M - (m0 + mk.wm) + 15) / 16;
      edge_nj = (N - (n0 + mk.wn) + 7) / 8;
      edge_mi = edge_mi < 0 ? 0 : (edge_mi > 4 ? 4 : edge_mi);
      edge_nj = edge_nj < 0 ? 0 : (edge_nj > 4 ? 4 : edge_nj);
    }
    // the skipping path runs only where it saves at least half of the warp's MMAs: its loads
    // are less well pipelined, and an edge warp that is slower per K step than its neighbours
    // holds the whole CTA's ring (measured: ragged cfg4 shapes 3-12% slower when every edge warp
    // took it; profiles/r02/ab_dmma_edge.txt)
    const bool interior = edge_mi * edge_nj > 8;
    for (int kt = kb; kt < ke; ++kt, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      if constexpr (FFMA) {
        // (a partial-step variant measured 3-5% slower on fp32 through code growth; the FFMA
        //  cases have K >= 750, where the tail is negligible)
        mk.stage(As + s * AL::STAGE, Bs + s * BL::STAGE);
      } else {
        const int krem = K - kt * BK;
        if (interior) {
          if (krem >= BK) mk.stage(As + s * AL::STAGE, Bs + s * BL::STAGE);
          else mk.stage_tail(As + s * AL::STAGE, Bs + s * BL::STAGE, (krem + 3) / 4);
        } else {
          mk.stage_edge(As + s * AL::STAGE, Bs + s * BL::STAGE, krem >= BK ? BK / 4 : (krem + 3) / 4,
                        edge_mi, edge_nj);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    if constexpr (kCsk) {
      if (sched.csplit) {
        consumers_sync();   // every consumer warp is done with the ring: it holds the partial
        double* part = reinterpret_cast<double*>(smem_raw);
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            part[mk.col(c) * kPP + mk.row(r)] = static_cast<double>(mk.value(r, c));
        cluster_sync_all();
        // rank r sums rows [r BM / S, (r + 1) BM / S) (S need not divide BM)
        const int S = sched.csplit;
        const uint32_t rank = cluster_rank();
        const int r0 = (int)rank * BM / S, RS = ((int)rank + 1) * BM / S - r0;
        for (int e = threadIdx.x; e < RS * BN; e += NCW * 32) {
          const int row = r0 + e % RS, col = e / RS;
          const uint32_t loc = smem_u32(part + col * kPP + row);
          double v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = q < S ? ld_dsmem(loc, (uint32_t)q) : 0.0;
          double sum = 0.0;
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q < S) sum += v[q];
          const int m = m0 + row, n = n0 + col;
          if (m < M && n < N) {
            T* q = C + (rC[m] + cC[n]);
            double out = alpha * sum;
            if (beta != 0.0) out = fma(beta, static_cast<double>(*q), out);
            store_c(q, static_cast<T>(out), false);
          }
        }
        cp_async_wait_all();
        cluster_sync_all();
        continue;
      }
    }
    // stream-K piece order: piece 0 (kb == 0) writes alpha*acc + beta*C; piece j >= 1 waits
    // for flag == j and adds alpha*acc; a piece that is not the last publishes flag = j + 1.
    const bool split = sk && !(kb == 0 && ke == sched.KT);
    int piece = 0;
    int* flag = nullptr;
    if (split) {
      const int s_local = tile - sched.D;
      const long long g_first = (long long)s_local * sched.KT;
      const int owner = sk_owner(sched, g_first);
      piece = blockIdx.x - owner;
      flag = flags + s_local;
      if (piece > 0) {
        if (threadIdx.x == 0) wait_flag(flag, (int)(sched.epoch | (unsigned)piece));
        consumers_sync();
      }
    }
    const bool accumulate = split && piece > 0;
    // (short K loops keep the load-add-store: with one or two K steps per piece the many
    //  concurrent reductions cost more at L2 than they save; f1 k32 682 -> 717 us with red,
    //  f2_07/08/10 -2..-6%; profiles/r02/ab_sk_red.txt)
    const bool red = TC_SK_RED && std::is_same<T, double>::value && sched.KT >= 8;
    const bool keep_c = split && ke < sched.KT;   // a later piece reads this tile back

    if constexpr (FFMA) {
      // FFMA epilogue through shared memory: the FFMA micro-kernel's thread layout puts a
      // lane's rows 4 apart (or 8), so direct stores would touch several times the sectors
      // they fill. The warp stages its 64 x 32 block as [n][m]; then consecutive lanes write
      // consecutive elements along C's unit-stride bundle (M: lane l takes rows l and l + 32
      // of every column; N: lane l takes column l, reading 4 rows per 16-byte load), one
      // 128-byte run per warp store when that bundle is contiguous. C is read the same way
      // when beta != 0 or for a stream-K accumulation.
      __syncwarp();
      if constexpr (A_VM) {   // rows 4 tm + {0..3} (+ 32): one 16-byte store per column
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float* d = epi + (mk.col(c) - mk.wn) * kEpiLD + (mk.row(0) - mk.wm);
          *reinterpret_cast<float4*>(d) =
              make_float4(mk.value(0, c), mk.value(1, c), mk.value(2, c), mk.value(3, c));
          *reinterpret_cast<float4*>(d + 32) =
              make_float4(mk.value(4, c), mk.value(5, c), mk.value(6, c), mk.value(7, c));
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int r = 0; r < 8; ++r)
            epi[(mk.col(c) - mk.wn) * kEpiLD + (mk.row(r) - mk.wm)] = mk.value(r, c);
      }
      cp_async_wait_all();
      __syncwarp();
      const bool read_c = accumulate || beta != 0.0;
      if (!c_lanes_n && !read_c && m0 + BM <= M && n0 + BN <= N) {
        // interior, write-only: no checks
        const IDX rca = wtab[lane], rcb = wtab[lane + 32];
#pragma unroll 8
        for (int j = 0; j < WN; ++j) {
          const IDX c = wtab[WM + j];
          const float* src = epi + j * kEpiLD;
          store_c(C + (rca + c), static_cast<T>(alpha * static_cast<double>(src[lane])), keep_c);
          store_c(C + (rcb + c), static_cast<T>(alpha * static_cast<double>(src[lane + 32])), keep_c);
        }
      } else if (!c_lanes_n) {
        const int ma = m0 + mk.wm + lane, mb = ma + 32;
        const IDX rca = wtab[lane], rcb = wtab[lane + 32];
        const bool ina = ma < M, inb = mb < M;
#pragma unroll 2
        for (int j0 = 0; j0 < WN; j0 += 8) {
          float olda[8], oldb[8];
          IDX cc[8];
          bool nin[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            cc[j] = wtab[WM + j0 + j];
            nin[j] = n0 + mk.wn + j0 + j < N;
            olda[j] = oldb[j] = 0.f;
            if (read_c) {
              if (ina && nin[j]) olda[j] = accumulate ? __ldcg(C + (rca + cc[j])) : C[rca + cc[j]];
              if (inb && nin[j]) oldb[j] = accumulate ? __ldcg(C + (rcb + cc[j])) : C[rcb + cc[j]];
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float* src = epi + (j0 + j) * kEpiLD;
            double va = alpha * static_cast<double>(src[lane]);
            double vb = alpha * static_cast<double>(src[lane + 32]);
            if (accumulate) { va += olda[j]; vb += oldb[j]; }
            else if (beta != 0.0) { va = fma(beta, (double)olda[j], va); vb = fma(beta, (double)oldb[j], vb); }
            if (ina && nin[j]) store_c(C + (rca + cc[j]), static_cast<T>(va), keep_c);
            if (inb && nin[j]) store_c(C + (rcb + cc[j]), static_cast<T>(vb), keep_c);
          }
        }
      } else {
        const int n = n0 + mk.wn + lane;
        const IDX cc = wtab[WM + lane];
        const bool nin = n < N;
#pragma unroll 2
        for (int i0 = 0; i0 < WM; i0 += 8) {
          float old[8];
          IDX rc[8];
          bool min_[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            rc[i] = wtab[i0 + i];
            min_[i] = m0 + mk.wm + i0 + i < M;
            old[i] = 0.f;
            if (read_c && nin && min_[i]) old[i] = accumulate ? __ldcg(C + (rc[i] + cc)) : C[rc[i] + cc];
          }
          const float4 x0 = *reinterpret_cast<const float4*>(epi + lane * kEpiLD + i0);
          const float4 x1 = *reinterpret_cast<const float4*>(epi + lane * kEpiLD + i0 + 4);
          const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            double v = alpha * static_cast<double>(xv[i]);
            if (accumulate) v += old[i];
            else if (beta != 0.0) v = fma(beta, (double)old[i], v);
            if (nin && min_[i]) store_c(C + (rc[i] + cc), static_cast<T>(v), keep_c);
          }
        }
      }
    } else if (TC_DMMA_STAGED && !c_lanes_n) {
      // DMMA epilogue through shared memory, 16 rows at a time: lanes 0-15 and 16-31 write 16
      // consecutive rows of two columns, i.e. two 128-byte runs per warp store when C is
      // unit-stride along M (the fragment layout gives four 64-byte pieces).
      cp_async_wait_all();
      const bool read_c = accumulate || beta != 0.0;
      const int ri = lane & 15, cp = lane >> 4;
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            epid[(mk.col(c) - mk.wn) * kEpiDLD + (mk.row(2 * pass + h) - mk.wm - 16 * pass)] =
                static_cast<double>(mk.value(2 * pass + h, c));
        __syncwarp();
        const int mrow = 16 * pass + ri;            // row within the warp block
        const bool min_ = m0 + mk.wm + mrow < M;
        const IDX rc = wtab[mrow];
#pragma unroll 2
        for (int j0 = 0; j0 < 16; j0 += 8) {
          double old[8];
          IDX cc[8];
          bool ok[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int col = 2 * (j0 + j) + cp;
            cc[j] = wtab[WM + col];
            ok[j] = min_ && n0 + mk.wn + col < N;
            old[j] = 0.0;
            if (read_c && ok[j]) {
              const T* q = C + (rc + cc[j]);
              old[j] = static_cast<double>(accumulate ? __ldcg(q) : *q);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int col = 2 * (j0 + j) + cp;
            double v = alpha * epid[col * kEpiDLD + ri];
            if (accumulate) v += old[j];
            else if (beta != 0.0) v = fma(beta, old[j], v);
            if (ok[j]) store_c(C + (rc + cc[j]), static_cast<T>(v), keep_c);
          }
        }
      }
    } else {

    // epilogue: C[rC[m] + cC[n]] = alpha*acc + beta*C (beta == 0: C not read); computed in
    // fp64, rounded once to T. C is read in chunks of 16 independent loads (two of the thread's
    // rows) so the loads of a chunk overlap instead of each waiting behind the previous store.
    cp_async_wait_all();
    __syncwarp();
    IDX cc[8];
    int nn[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      nn[c] = n0 + mk.col(c);
      cc[c] = wtab[WM + mk.col(c) - mk.wn];
    }
    const bool read_c = accumulate || beta != 0.0;
    if (red && accumulate) {
      // stream-K accumulation at L2 (red_add_c): no reads, no round trips
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int m = m0 + mk.row(r);
        const IDX rcr = wtab[mk.row(r) - mk.wm];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (m < M && nn[c] < N)
            red_add_c(reinterpret_cast<double*>(C + (rcr + cc[c])),
                      alpha * static_cast<double>(mk.value(r, c)));
      }
    } else if (!read_c && m0 + BM <= M && n0 + BN <= N) {
      // interior tile, C write-only: no bounds checks, no reads, all offsets up front (the
      // common case of small-K contractions, where the epilogue is most of the work)
      IDX rc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) rc[r] = wtab[mk.row(r) - mk.wm];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          store_c(C + (rc[r] + cc[c]), static_cast<T>(alpha * static_cast<double>(mk.value(r, c))),
                  keep_c);
    } else
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) {
      int mm[2];
      IDX rc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mm[h] = m0 + mk.row(2 * r2 + h);
        rc[h] = wtab[mk.row(2 * r2 + h) - mk.wm];
      }
      double old[2][8];
      if (read_c) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            old[h][c] = 0.0;
            if (mm[h] < M && nn[c] < N) {
              const T* q = C + (rc[h] + cc[c]);
              old[h][c] = static_cast<double>(accumulate ? __ldcg(q) : *q);
            }
          }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (mm[h] >= M) continue;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (nn[c] >= N) continue;
          double v = alpha * static_cast<double>(mk.value(2 * r2 + h, c));
          if (accumulate) v += old[h][c];
          else if (beta != 0.0) v = fma(beta, old[h][c], v);
          store_c(C + (rc[h] + cc[c]), static_cast<T>(v), keep_c);
        }
      }
    }
    }   // DMMA epilogue
    if (split) {
      // publish this piece (epoch-tagged: nothing is reset for the next launch)
      consumers_sync();
      if (threadIdx.x == 0) {
        __threadfence();
        if (ke < sched.KT) st_release(flag, (int)(sched.epoch | (unsigned)(piece + 1)));
      }
    }
  }
}


// Work weights of a ragged stream-K tail (Sched::weighted): a tile's time per K step is its
// busiest SMSP's MMA count -- the two consumer warps of an SMSP (dmma_wm / dmma_wn), each doing
// all 16 of its m16n8 blocks, or only the mi x nj that hold data when that is at most half
// (the stage_edge rule) -- clamped to >= 1/4 of a full tile so no CTA's range is empty.
// TC_SK_WEIGHTS=0 turns it off (read per call).
inline void set_tile_weights(Sched& sc, int M, int N, int tiles_m, int tiles_n) {
  const int n = sc.T - sc.D;
  const char* e = getenv("TC_SK_WEIGHTS");
  sc.weighted = 0;
  // long K loops only: on short ones (cfg1, 12 us) the moved boundaries cost more than the
  // balance gains (12.0 -> 14.5 us; f2_17 1034.6 -> 988.2 us, profiles/r02/ab_sk_weights.txt)
  if (sc.P_sk == 0 || n > kMaxWeighted || sc.KT < 256 || (M % BM == 0 && N % BN == 0) ||
      (e && *e == '0'))
    return;
  sc.cum[0] = 0;
  bool any = false;
  for (int i = 0; i < n; ++i) {
    int tm, tn;
    tile_coords<GROUP_M>(sc.D + i, tiles_m, tiles_n, &tm, &tn);
    int smsp[4] = {0, 0, 0, 0};
    for (int w = 0; w < NCW; ++w) {
      int mi = (M - (tm * BM + dmma_wm(w)) + 15) / 16, nj = (N - (tn * BN + dmma_wn(w)) + 7) / 8;
      mi = mi < 0 ? 0 : (mi > 4 ? 4 : mi);
      nj = nj < 0 ? 0 : (nj > 4 ? 4 : nj);
      smsp[w & 3] += mi * nj > 8 ? 16 : mi * nj;
    }
    int wt = 0;
    for (int q = 0; q < 4; ++q) wt = smsp[q] > wt ? smsp[q] : wt;
    wt = wt < 8 ? 8 : wt;
    any = any || wt < 32;
    sc.cum[i + 1] = sc.cum[i] + wt;
  }
  sc.weighted = any ? 1 : 0;
}

// Cluster split-K instead of the stream-K schedule (Sched::csplit) where the stream-K split
// would chain >= 4 pieces per tile (every tile in the tail): the largest S in 8 .. 4 (16 .. 4,
// non-portable, for short pieces) whose T clusters are co-resident in one wave (clusters must
// sit inside a GPC: at 227 KB per CTA only 15 clusters of 8, 22 of 6 and 33 of 4 fit on a B200,
// so 16 tiles in clusters of 8 take two waves) and whose T S CTAs cover >= 80% (short pieces:
// 40%) of the CTAs stream-K would run, with >= 2 K steps per CTA. TC_CSK=0 turns it off (read
// per call).
template <typename K>
inline int max_active_clusters(K kern, int S, int smem, std::atomic<int> (*cache)[17]) {
  // cache: the caller's, one per kernel instantiation (by device and S = 1 .. 16); the
  // non-portable attribute below is set per kernel as well
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices || S < 1 || S > 16)
    return 0;
  const int i = S;
  int v = cache[dev][i].load(std::memory_order_relaxed);
  if (v > 0) return v - 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)S;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (S > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                   cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[dev][i].store(n + 1, std::memory_order_relaxed);
  return n;
}

template <typename T, bool A_VM, bool B_VK, typename IDX, bool FFMA, typename Kern>
inline int csk_split(const Sched& sc, int nsm, bool allow, Kern kern, int smem,
                     std::atomic<int> (*cache)[17]) {
  if constexpr (!csk_fits<T, A_VM, B_VK, IDX, FFMA>()) {
    return 0;
  } else {
    const char* e = getenv("TC_CSK");
    if (!allow || (e && *e == '0') || sc.D != 0 || sc.P_sk < 4 * sc.T) return 0;
    // Short stream-K pieces (<= 64 K steps per CTA): the chain of fix-ups per tile, not the
    // arithmetic, sets the time, so cluster split-K pays even on fewer SMs: coverage >= 40% and
    // non-portable clusters up to 16 (323^2 x 3000 0.34 -> 0.73 of DGEMM, 384^2 x 4096 0.42 ->
    // 0.69). Long pieces keep >= 80% and S <= 8 (at 40%, f2_16 / f2_17 with K = 104329 fell
    // 0.77 -> 0.43, 0.89 -> 0.46; profiles/r02/ab_csk_sizes.txt). TC_CSK_COV / _MAX override.
    const bool short_pieces = (long long)sc.T * sc.KT <= 64LL * sc.P_sk;
    const char* em = getenv("TC_CSK_MAX");
    const int smax = em && atoi(em) >= 4 && atoi(em) <= 16 ? atoi(em) : short_pieces ? 16 : 8;
    // S in {smax, 7, 6, 5, 4}: a cluster size that is not a power of two lets a few-tile shape
    // whose T clusters of 8 do not fit in one wave still spread its tiles over most SMs (fp64
    // 512^3: 16 clusters of 8 or 7 do not fit, 16 of 6 do; TC_CSK_POW2=1: {smax, 4} only, the
    // earlier policy; profiles/r02/ab_csk_sizes.txt)
    const char* ec = getenv("TC_CSK_COV");
    const int cov = ec && atoi(ec) > 0 ? atoi(ec) : short_pieces ? 40 : 80;
    const char* ep = getenv("TC_CSK_POW2");
    const bool pow2 = ep && *ep == '1';
    for (int S = smax; S >= 4; S = pow2 ? (S > 8 ? 8 : S / 2) : S - 1)
      if (sc.T * S <= nsm && sc.KT >= 2 * S && 100 * sc.T * S >= cov * sc.P_sk &&
          sc.T <= max_active_clusters(kern, S, smem, cache))
        return S;
    return 0;
  }
}

template <typename T, typename IDX, bool A_VM, bool B_VK, int A_MODE, int B_MODE, bool FFMA>
int launch(const LaunchArgs& a, cudaStream_t stream) {
  constexpr int STAGES = ring_stages<T, A_VM, B_VK, IDX, FFMA>();
  constexpr int smem = smem_bytes<T, A_VM, B_VK, IDX, FFMA>(STAGES);
  auto kern = tc_dmma_ws_kernel<T, IDX, A_VM, B_VK, A_MODE, B_MODE, FFMA>;
  static std::atomic<int> attr[kMaxDevices];
  if (!ensure_dyn_smem(kern, smem, attr)) return -1;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int KT = (a.K + BK - 1) / BK;
  // every partial wave goes to the stream-K tail (threshold 101%): since the fix-ups add at L2
  // (red.global.add) a split tail beats a nearly full data-parallel wave (cfg4_11 fp64 +3.8%,
  // cfg4_12 +1.2%, geomean over cfg4 fp64 / f1 / f2 +0.07%; round 1's 88% was measured with
  // load-add-store fix-ups; profiles/r02/ab_dppct.txt). TC_WS_DPPCT overrides (measurement).
  static const int dp_pct = [] {
    const char* e = getenv("TC_WS_DPPCT");
    return e ? atoi(e) : 101;
  }();
  // up to 48 stream-K pieces per tile: few-tile, long-K shapes then keep every SM busy (this
  // kernel's fix-up links are cheap: 256^2 x 65536 0.39 -> 0.52, 128^2 x 262144 0.12 -> 0.27 of
  // DGEMM; profiles/r01/ab_max_pieces.txt)
  const char* msk = getenv("TC_WS_MINSK");   // measurement override of kMinSkIters (per call)
  const int min_sk = msk && atoi(msk) > 0 ? atoi(msk) : kMinSkIters;
  Sched sc = make_sched(tiles_m * tiles_n, KT, a.num_sms, a.stream_k, dp_pct, min_sk, 48);
  if (sc.P_sk > 0 && (sc.T - sc.D) > a.flags_cap) {   // cannot happen: S < 2 * num_sms
    Sched dp = make_sched(tiles_m * tiles_n, KT, a.num_sms, false);
    sc = dp;
  }
  if (!FFMA && TC_DMMA_EDGE) set_tile_weights(sc, a.M, a.N, tiles_m, tiles_n);
  int* flags = a.flags;
  sc.epoch = a.flag_epoch;
  int grid = sc.D > 0 ? sc.P : sc.P_sk;
  static std::atomic<int> csk_cache[kMaxDevices][17];
  const int S = csk_split<T, A_VM, B_VK, IDX, FFMA>(sc, a.num_sms, a.stream_k, kern, smem,
                                                    csk_cache);
  if (S > 0) {
    Sched cs = make_sched(sc.T, KT, a.num_sms, false);
    cs.csplit = S;
    cs.epoch = a.flag_epoch;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sc.T * S));
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (getenv("TC_CSK_DEBUG")) {
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      fprintf(stderr, "csk: T %d S %d KT %d max active clusters %d\n", sc.T, S, KT, ncl);
    }
    if (cudaLaunchKernelEx(&cfg, kern, static_cast<const T*>(a.A), static_cast<const T*>(a.B),
                           static_cast<T*>(a.C), static_cast<const IDX*>(a.rA),
                           static_cast<const IDX*>(a.cA), static_cast<const IDX*>(a.rB),
                           static_cast<const IDX*>(a.cB), static_cast<const IDX*>(a.rC),
                           static_cast<const IDX*>(a.cC), a.vA, a.vB, a.M, a.N, a.K, tiles_m,
                           tiles_n, a.alpha, a.beta, cs, flags, a.c_lanes_n) != cudaSuccess)
      return -1;
    return 1;
  }
  // wave alignment only pays when a tile's K panels are long enough for L2 sharing to matter;
  // with short K loops the per-wave wait is pure overhead (f1 k5: 15% of samples at the barrier)
  sc.wave_sync = a.wave_sync && a.wave_base != nullptr && sc.D >= 2 * sc.P && KT >= 64;
  if (sc.wave_sync) {
    // every whole tile adds one to the device counter
    sc.wave_base = a.wave_base->fetch_add((unsigned)sc.D, std::memory_order_relaxed);
  }
  kern<<<grid, NTHREADS, smem, stream>>>(
      static_cast<const T*>(a.A), static_cast<const T*>(a.B), static_cast<T*>(a.C),
      static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.vA, a.vB, a.M, a.N, a.K,
      tiles_m, tiles_n, a.alpha, a.beta, sc, flags, a.c_lanes_n);
  if (cudaPeekAtLastError() != cudaSuccess) return -1;
  return 1;
}

template <typename T, typename IDX, int A_MODE, int B_MODE, bool FFMA>
int dispatch_dir(const LaunchArgs& a, cudaStream_t s) {
  if (a.a_vec_m)
    return a.b_vec_k ? launch<T, IDX, true, true, A_MODE, B_MODE, FFMA>(a, s)
                     : launch<T, IDX, true, false, A_MODE, B_MODE, FFMA>(a, s);
  return a.b_vec_k ? launch<T, IDX, false, true, A_MODE, B_MODE, FFMA>(a, s)
                   : launch<T, IDX, false, false, A_MODE, B_MODE, FFMA>(a, s);
}

// All B gather modes for one A mode (each A mode is instantiated in its own translation unit).
template <typename T, bool FFMA, int A_MODE>
int dispatch_b(const LaunchArgs& a, cudaStream_t s) {
  switch (a.b_mode) {
    case 0: return dispatch_dir<T, int, A_MODE, 0, FFMA>(a, s);
    case 1: return dispatch_dir<T, int, A_MODE, 1, FFMA>(a, s);
    default: return dispatch_dir<T, int, A_MODE, 2, FFMA>(a, s);
  }
}

// fp32, A and B both gathered along K: A through the transposing gather (mode 3) into the
// [k][m] layout, so the consumer runs PAIR_R.
template <typename T, bool FFMA>
int dispatch_a_transposed(const LaunchArgs& a, cudaStream_t s) {
  switch (a.b_mode) {
    case 0: return launch<T, int, true, true, 3, 0, FFMA>(a, s);
    case 1: return launch<T, int, true, true, 3, 1, FFMA>(a, s);
    default: return launch<T, int, true, true, 3, 2, FFMA>(a, s);
  }
}

// 64-bit offsets: per-vector gathers only (the element gather keeps 16 offsets per thread).
template <typename T, bool FFMA>
int dispatch_idx64(const LaunchArgs& a, cudaStream_t s) {
  return dispatch_dir<T, long long, 1, 1, FFMA>(a, s);
}

}  // namespace ws
}  // namespace tcb
