// fp32 contraction on the 5th-generation tensor cores (sm_100a tcgen05, kind::tf32) with the
// 3xTF32 split: every fp32 operand x is split into hi = tf32(x) and lo = x - hi, and
// A.B = Ahi.Bhi + Ahi.Blo + Alo.Bhi (the Alo.Blo term, ~2^-20 relative, is dropped), accumulated
// in fp32 in tensor memory in chunks of K summed with rounded fp32 adds (reading R18 in
// DESIGN.md). Normwise error <= 7e-7 on cfg4 at full size (FFMA2 kernel: <= 1.1e-6), against the
// 1e-5 bound of BASELINE north_star checked by the parity tests.
//
// The paper's method is unchanged: the tiles are gathered from the tensors' strides through the
// scatter vectors -- here straight into the tensor cores' canonical
// shared-memory layout, or for A on into tensor memory -- and C is written through its scatter
// vectors with alpha / beta. One CTA per SM walks the persistent schedule of
// sched.cuh (whole 128 x 128 tiles of C, then stream-K pieces fixed up in place). Default build
// (A in TMEM, N = 128 MMAs, one K step per chunk):
//   warps 0-3   producers: cp.async gathers of A and B (128 x 32 each per K step) into the stage:
//               4-byte element copies laid out so a warp instruction reads whole 32-byte
//               sectors of a contiguous operand (8 rows x 4 K or 4 rows x 8 K), or 16-byte
//               vector copies where the plan proved the operand's vectors contiguous and aligned
//   warps 4-7   converters: B's lo = x - trunc(x) next to B's raw value (the tensor core
//               reads hi as the raw value's tf32 bits, i.e. truncated); A's hi and lo go to an
//               A slot in tensor memory (one row per thread, tcgen05.st)
//   warps 8-11  epilogue: tcgen05.ld of each chunk accumulator (warp w reads TMEM lanes
//               32 (w - 8)..), added into the running sum in TMEM; at the end of a work item
//               one row of C per thread, alpha * acc + beta * C through rscat_C / cscat_C
//   warp 12     MMA issuer: one lane issues 3 x 4 tcgen05.mma (M = N = 128, K = 8, A from TMEM)
//               per K step and commits them to the stage's, the A slot's and the chunk's
//               barriers; two TMEM chunk accumulators let the epilogue's adds overlap the next
//               chunk's MMAs.
// Compile-time forms of the same source: TC_UMMA_N256 (umma_f32_n256.cu), TC_UMMA_PAIR
// (umma_f32_pair.cu); measurement switches: TC_UMMA_TMEM_A, TC_UMMA_CHUNK, TC_UMMA_PW/CW,
// TC_UMMA_HI_TRUNC, TC_UMMA_TRACE, TC_UMMA_PROF.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"
#include "sched.cuh"

// This file is compiled three times: as itself (N = 128 MMAs, one K step per chunk), through
// umma_f32_n256.cu (N = 256 form, four K steps per chunk, element gathers only) and through
// umma_f32_pair.cu (CTA pairs), each in its own namespace with its own launch entry.
#ifndef TC_UMMA_NS
#define TC_UMMA_NS umma
#define TC_UMMA_LAUNCH launch_umma_f32
#endif

namespace tcb {
namespace TC_UMMA_NS {

using namespace dev;
using namespace sched;

// A operand in tensor memory (TC_UMMA_TMEM_A=1): the converter warps write A's hi and lo to TMEM
// with tcgen05.st (lane = row of A, one column per k) and the MMAs take A from there, so A's lo
// never goes to shared memory and the tensor core reads only B from it; the freed shared memory
// buys a fourth stage. Off: A hi and lo are staged in shared memory like B.
#ifndef TC_UMMA_TMEM_A
#define TC_UMMA_TMEM_A 1
#endif
constexpr bool kTmemA = TC_UMMA_TMEM_A;
constexpr int BM = 128, BN = 128, BK = 32, STAGES = kTmemA ? 4 : 3;
#ifndef TC_UMMA_PW
#define TC_UMMA_PW 4
#endif
constexpr int kPW = TC_UMMA_PW;            // producer warps (4 or 8)
#ifndef TC_UMMA_CW
#define TC_UMMA_CW 4
#endif
constexpr int kCW = TC_UMMA_CW;            // converter warps (4 or 8; 8: two per TMEM lane quarter)
constexpr int kConv0 = kPW, kEpi0 = kPW + kCW, kMmaW = kEpi0 + 4;   // first warp of each role
constexpr int kThreads = (kMmaW + 1) * 32;
constexpr int kTile = (BK / 4) * (128 * 4 + 16);   // floats per operand tile (padded K chunks)
// N = 256 form (TC_UMMA_N256=1, needs A in TMEM): per K = 8 one 128x256 MMA of A hi against
// [B hi; B lo] (256 rows: hi rows, then lo rows, in every K chunk) gives Ahi.Bhi in accumulator
// columns 0-127 and Ahi.Blo in 128-255, and one 128x128 MMA adds Alo.Bhi to columns 128-255:
// two MMAs instead of three, and a 128x256 MMA costs about what a 128x128 one does
// (tools/calib/umma_rate_test.cu: ~145 cycles each).
#ifndef TC_UMMA_N256
#define TC_UMMA_N256 0
#endif
constexpr bool kN256 = TC_UMMA_N256 && kTmemA;
// CTA-pair form (TC_UMMA_PAIR=1, N = 128 form with A in TMEM): two CTAs of a cluster run one
// 256 x 128 tile with tcgen05.mma.cta_group::2 (M = 256) issued by the leader; each CTA stages its
// 128 rows of A (in its own TMEM) and half of B (64 rows), so one MMA instruction does twice the
// work and each SM gathers and converts a quarter less.
#ifndef TC_UMMA_PAIR
#define TC_UMMA_PAIR 0
#endif
constexpr bool kPair = TC_UMMA_PAIR && kTmemA && !kN256;
constexpr int kRowsB = kPair ? 64 : 128;    // B rows (N) staged per CTA
constexpr int kTM = kPair ? 256 : 128;      // rows of C per tile
constexpr int kChunkB = kN256 ? 2 * 128 * 4 + 16 : kRowsB * 4 + 16;   // B's K-chunk stride (floats)
constexpr int kTileB = (BK / 4) * kChunkB;
// stage layout: [A hi (raw), A lo, B hi (raw), B lo], or [A raw, B hi (raw), B lo] with A in TMEM,
// or [A raw, B (hi and lo rows interleaved per K chunk)] in the N = 256 form
constexpr int kStage = kTmemA ? kTile + (kN256 ? kTileB : 2 * kTileB) : 4 * kTile;
constexpr int kOffAl = kTile, kOffBh = kTmemA ? kTile : 2 * kTile, kOffBl = kOffBh + kTileB;
constexpr int GROUP_M = 2;
// The tensor core's fp32 accumulation is biased (it truncates): on one-signed data the relative
// error grows with the number of MMAs chained into one accumulator (3xTF32, K = 128 per
// accumulator: -2.6e-6 bias; K = 32: -7.6e-7), so the accumulator restarts every kChunkSteps K
// steps and the epilogue warps add each chunk into a running sum held in TMEM (rounded fp32
// adds, like an FFMA loop). One K step per chunk costs ~2% against four
// (profiles/r01/ab_umma_chunk.txt).
#ifndef TC_UMMA_CHUNK
#define TC_UMMA_CHUNK 1
#endif
constexpr int kChunkSteps = TC_UMMA_CHUNK;   // K steps of BK per chunk
// TMEM (512 columns): kChunkBufs chunk accumulators of BN columns, then the running sum; three
// buffers give the epilogue two chunks of slack while it stores a finished tile
// (two with A in TMEM, whose two 64-column slots -- hi, lo -- take the last 128 columns)
// (N = 256 form: one 256-column chunk accumulator, released as soon as the epilogue has read it)
constexpr int kChunkBufs = kN256 ? 1 : (kTmemA ? 2 : 3);
constexpr int kChunkCols = kN256 ? 2 * BN : BN;
constexpr int kSumCol = kChunkBufs * kChunkCols;
constexpr int kACol = kSumCol + BN, kASlots = 2;
// shared memory: stage ring, barriers, then the epilogue's transpose buffer (32 x 33 floats per
// epilogue warp) for read-modify-writes of a C whose unit stride runs along N
constexpr int kBarBytes = (3 * STAGES + 2 * kChunkBufs + kASlots) * 8 + 16;
constexpr int kEpiOff = (STAGES * kStage * 4 + kBarBytes + 127) / 128 * 128;
constexpr int kSmemBytes = kEpiOff + 4 * 32 * 33 * 4;
static_assert(kSumCol + BN + (kTmemA ? kASlots * 2 * BK : 0) <= 512, "TMEM columns");

__device__ __forceinline__ uint32_t tmem_u32_addr(const void* p) { return smem_u32(p); }

// Canonical SWIZZLE_NONE K-major layout (in floats): core matrix = 8 rows x 4 K (16 B per row);
// row groups of 8 at 32 floats (SBO 128 B), K chunks of 4 at kChunk floats (LBO); one K = 8 MMA
// step spans two K chunks. kChunk = 512 + 16: the 64-byte pad puts the two K chunks a K-run
// gather writes in one instruction on different banks. (The MN-major tf32 operand mode left the
// accumulator at zero on this part, tools/calib/umma_tf32_test.cu, so both operands are K-major.)
constexpr int kChunk = 128 * 4 + 16;
// K chunk stride of an operand's staging (floats): the one-row-per-instruction K gather (mode 7)
// writes eight consecutive chunks per instruction, which a 64-byte pad would put on two bank
// groups; a 16-byte pad spreads them over all banks
// (the same pad under the 16-byte K-vector gathers, mode 2, removes their bank conflicts but
// measured 1% slower over cfg4: profiles/r02/ab_umma_vkpad.txt)
template <int BASE, int MODE> constexpr int chunk_stride() {
  return BASE + ((MODE == 7 || MODE == 5) ? 4 : 16);
}
template <int CH = kChunk>
__device__ __forceinline__ int tile_off(int r, int k) {
  return (k >> 2) * CH + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}

template <int CH = kChunk>
__device__ __forceinline__ uint64_t make_desc(const float* base, int j) {   // MMA step j (K 8j..)
  const uint32_t addr = smem_u32(base + j * 2 * CH);
  const uint32_t lbo = CH * 4, sbo = 128;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  return d;                                     // SWIZZLE_NONE, base offset 0
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&u)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&u)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n"
      :: "r"(taddr), "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]),
         "r"(u[6]), "r"(u[7]), "r"(u[8]), "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]),
         "r"(u[13]), "r"(u[14]), "r"(u[15]), "r"(u[16]), "r"(u[17]), "r"(u[18]), "r"(u[19]),
         "r"(u[20]), "r"(u[21]), "r"(u[22]), "r"(u[23]), "r"(u[24]), "r"(u[25]), "r"(u[26]),
         "r"(u[27]), "r"(u[28]), "r"(u[29]), "r"(u[30]), "r"(u[31])
      : "memory");
}
#ifndef TC_UMMA_HI_TRUNC
#define TC_UMMA_HI_TRUNC 1
#endif
template <int N>
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&u)[N]) {
  static_assert(N == 16, "x16");
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};\n"
      :: "r"(taddr), "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]),
         "r"(u[6]), "r"(u[7]), "r"(u[8]), "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]),
         "r"(u[13]), "r"(u[14]), "r"(u[15])
      : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t taddr, const uint32_t (&u)[N]) {
  if constexpr (N == 32) tmem_st32(taddr, u);
  else tmem_st16(taddr, u);
}
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
#ifndef TC_UMMA_LO_RNA
#define TC_UMMA_LO_RNA 0   // 1: lo rounded to tf32 (0: the tensor core truncates it; +11%, bias 7.6e-7 -> 9.6e-7)
#endif
__device__ __forceinline__ float tf32_rna(float x);
__device__ __forceinline__ float lo_round(float x) {
#if TC_UMMA_LO_RNA
  return tf32_rna(x);
#else
  return x;
#endif
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// Producer side of one operand X (A: rows = M, B: rows = N), 4-byte cp.async element gathers
// laid out so that a warp instruction touches as few 32-byte sectors as the operand allows:
//  KR = false (X contiguous along its rows): lanes = 8 rows x 4 K, one core matrix per
//             instruction, 32-byte runs along the rows
//  KR = true  (X contiguous along K): lanes = 4 rows x 8 K, 32-byte runs along K (two core
//             matrices half-filled, on disjoint banks thanks to the K-chunk pad)
// Either way 4 sectors per 128 bytes when the operand is contiguous (a K-run operand read with
// the row mapping would touch 8).
template <typename IDX, bool KR, int CH = kChunk, int ROWS = 128>
struct Gather {
  static constexpr int RG = KR ? 4 : 8;               // rows per instruction
  static constexpr int KG = KR ? 8 : 4;               // K per instruction
  static constexpr int NR = ROWS / RG / kPW;          // row groups per warp
  static constexpr int NK = BK / KG;                  // K groups per stage
  IDX ro[NR];
  uint32_t rv;
  IDX ko[NK];
  __device__ __forceinline__ static int row(int w, int i, int l) {
    return RG * (w * NR + i) + (KR ? (l >> 3) : (l >> 2));
  }
  __device__ __forceinline__ static int kin_(int j, int l) {
    return KG * j + (KR ? (l & 7) : (l & 3));
  }
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    rv = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int r = base + row(w, i, l);
      ro[i] = rtab[r];                       // tables are padded past the extent
      rv |= (r < extent ? 1u : 0u) << i;
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
#pragma unroll
    for (int j = 0; j < NK; ++j) ko[j] = __ldg(ktab + k0 + kin_(j, l));
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      const int kk = kin_(j, l);
      const bool kin = k0 + kk < K;
#pragma unroll
      for (int i = 0; i < NR; ++i)
        cp_async4(sm + tile_off<CH>(row(w, i, l), kk), g + (ro[i] + ko[j]), kin && ((rv >> i) & 1u));
    }
  }
};

// 16-byte vector gathers (the block-scatter decision of P:644-683 at 4-float granularity), used
// when the plan proved every vector of the operand contiguous and 16-byte aligned (a_vec_all /
// b_vec_all): a quarter of the copy instructions of the element gathers.
//  GatherVK: vectors along K (4 consecutive k of one row) into the K-major staging layout;
//            lanes = 4 rows x 8 vectors, i.e. 4 full 128-byte runs per instruction
//  GatherVM: vectors along the rows (A only: 4 consecutive m at one k) into a [k][m] staging
//            layout (row k = 128 floats) that the converter warps read column-wise into TMEM;
//            one instruction = one k, 128 consecutive m
template <typename IDX, int CH = kChunk, int ROWS = 128>
struct GatherVK {
  static constexpr int NR = ROWS / 4 / kPW;          // row groups of 4 per warp
  IDX ro[NR];
  uint32_t rv;
  IDX ko;
  __device__ __forceinline__ static int row(int w, int i, int l) { return 4 * (w * NR + i) + (l >> 3); }
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    rv = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int r = base + row(w, i, l);
      ro[i] = rtab[r];
      rv |= (r < extent ? 1u : 0u) << i;
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    ko = __ldg(ktab + k0 + 4 * (l & 7));
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
    const int kk = 4 * (l & 7);
    const bool kin = k0 + kk < K;                    // K is a multiple of 4 here
#pragma unroll
    for (int i = 0; i < NR; ++i)
      cp_async16(sm + tile_off<CH>(row(w, i, l), kk), g + (ro[i] + ko), kin && ((rv >> i) & 1u));
  }
};

template <typename IDX>
struct GatherVM {
  static constexpr int NKW = BK / kPW;               // k rows per warp
  IDX ro;
  bool rv;
  IDX ko[NKW];
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    const int r = base + 4 * l;
    ro = rtab[r];
    rv = r < extent;                                 // M is a multiple of 4 here
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    const int w = (threadIdx.x >> 5);
#pragma unroll
    for (int j = 0; j < NKW; ++j) ko[j] = __ldg(ktab + k0 + w * NKW + j);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < NKW; ++j) {
      const int k = w * NKW + j;
      cp_async16(sm + k * BM + 4 * l, g + (ro + ko[j]), rv && k0 + k < K);
    }
  }
};

// 8-byte pair gathers (the block-scatter decision at 2-float granularity, a_vec2_all /
// b_vec2_all): where the 16-byte vectors of an operand are not all contiguous and aligned but its
// pairs are (odd lengths break vectors of four more often than pairs: 26 of cfg4's 40 operands
// qualify against 17), half the copy instructions of the element gathers -- the producers of the
// element-gather cases issue one 4-byte cp.async per element and are bound by that (~8 cycles
// each, profiles/r02/umma_prof_roles.txt).
//  GatherP2K: pairs along K into the K-major staging layout (a pair never straddles a
//             core-matrix row)
//  GatherP2M: pairs along the rows (A only) into the [k][m] staging of GatherVM; lanes = 32 pairs
//             = 64 consecutive m at one k
template <typename IDX, int CH = kChunk, int ROWS = 128>
struct GatherP2K {
  // lanes = 2 rows x 16 pairs (all 32 K of a step): two 128-byte lines per instruction when
  // the rows' K runs are contiguous (4 rows x 8 pairs touched four); K chunks 16 bytes apart
  // mod 128 (chunk_stride), so the eight chunks of a row land on distinct banks. The warp's 32
  // row offsets live one per lane and are shuffled to the instruction that needs them.
  static constexpr int NRW = ROWS / kPW;             // rows per warp
  static_assert(NRW == 32, "one row offset per lane");
  IDX rl;
  uint32_t rv;
  IDX ko;
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    const int r = base + NRW * w + l;
    rl = rtab[r];
    rv = __ballot_sync(0xffffffffu, r < extent);
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    ko = __ldg(ktab + k0 + 2 * (l & 15));
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
    const int kk = 2 * (l & 15);
    const bool kin = k0 + kk < K;                    // K is even here
#pragma unroll
    for (int i = 0; i < NRW / 2; ++i) {
      const int r = 2 * i + (l >> 4);
      const IDX ro = __shfl_sync(0xffffffffu, rl, r);
      cp_async8(sm + tile_off<CH>(NRW * w + r, kk), g + (ro + ko), kin && ((rv >> r) & 1u));
    }
  }
};

template <typename IDX>
struct GatherP2M {
  static constexpr int NKW = BK / kPW;               // k rows per warp
  IDX ro[2];
  bool rv[2];
  IDX ko[NKW];
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = base + 64 * h + 2 * l;
      ro[h] = rtab[r];
      rv[h] = r < extent;                            // M is even here
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    const int w = (threadIdx.x >> 5);
#pragma unroll
    for (int j = 0; j < NKW; ++j) ko[j] = __ldg(ktab + k0 + w * NKW + j);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < NKW; ++j) {
      const int k = w * NKW + j;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        cp_async8(sm + k * BM + 64 * h + 2 * l, g + (ro[h] + ko[j]), rv[h] && k0 + k < K);
    }
  }
};

// Element gathers with one line per warp instruction where the operand allows it. The 8 x 4 and
// 4 x 8 lane mappings above fill whole 32-byte sectors of a contiguous operand but touch four
// 128-byte lines per instruction, and where the traversal interleaves dimensions (R17
// sub-division) up to 16; an L1 line costs ~2 cycles per instruction (B300_MICROARCH), and these
// gathers are what bounds the producer warps (profiles/r02/umma_prof_roles.txt). Counted by
// sampling cfg4's 40 operands: 208 lines per 40 instructions with the mappings above, 99 with
//  GatherK32: lanes = 32 consecutive K entries of one row (operands gathered along K); the row's
//             offset is shuffled from the lane that holds it; K chunks 16 bytes apart mod 128 so
//             the eight 16-byte chunks an instruction writes land on distinct banks
//  GatherR32: lanes = 32 consecutive rows at one k (operands gathered along their rows); the
//             K offset is shuffled from the lane that holds it
template <typename IDX, int CH = kChunk, int ROWS = 128>
struct GatherK32 {
  static constexpr int NRW = ROWS / kPW;             // rows per warp
  static_assert(NRW == 32, "one row per lane of the offset register");
  IDX rl;                                            // offset of row 32 w + lane
  uint32_t rv;                                       // row validity, one bit per row of the warp
  IDX ko;                                            // offset of K entry k0 + lane
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    const int r = base + NRW * w + l;
    rl = rtab[r];                                    // tables are padded past the extent
    rv = __ballot_sync(0xffffffffu, r < extent);
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    ko = __ldg(ktab + k0 + l);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
    const bool kin = k0 + l < K;
#pragma unroll
    for (int i = 0; i < NRW; ++i) {
      const IDX ro = __shfl_sync(0xffffffffu, rl, i);
      cp_async4(sm + tile_off<CH>(NRW * w + i, l), g + (ro + ko), kin && ((rv >> i) & 1u));
    }
  }
};

template <typename IDX, int CH = kChunk, int ROWS = 128>
struct GatherR32 {
  static constexpr int NRW = ROWS / kPW;             // rows per warp
  static_assert(NRW == 32, "one row per lane");
  IDX ro;                                            // offset of row 32 w + lane
  bool rv;
  IDX kl;                                            // offset of K entry k0 + lane
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    const int r = base + NRW * w + l;
    ro = rtab[r];
    rv = r < extent;
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    kl = __ldg(ktab + k0 + l);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const IDX ko = __shfl_sync(0xffffffffu, kl, k);
      cp_async4(sm + tile_off<CH>(NRW * w + l, k), g + (ro + ko), rv && k0 + k < K);
    }
  }
};

// B gathered along N with 16-byte vectors / 8-byte pairs (N = 256 form only, modes 10 / 11): B's
// K-major layout keeps consecutive n 16 bytes apart, so N vectors cannot land in it directly;
// they go to a [k][n] staging that occupies the lo half of each K chunk (rows 128-255 x 4 K =
// 512 floats, the same size), and the converter warps move them into the hi rows and write the
// lo rows over the staging (all values read into registers first). A quarter (vectors) or half
// (pairs) of the element gathers' copy instructions for B (19 of cfg4's 40 operands have N pairs).
template <typename IDX, int CH, int VEC>
struct GatherVN {
  static constexpr int KPW = BK / kPW;               // k rows per warp (8)
  static constexpr int NPL = 32 * VEC;               // n per warp instruction (128 / 64)
  IDX ro[128 / NPL];
  bool rv[128 / NPL];
  IDX ko[KPW];
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
#pragma unroll
    for (int h = 0; h < 128 / NPL; ++h) {
      const int r = base + NPL * h + VEC * l;
      ro[h] = rtab[r];
      rv[h] = r < extent;                            // N is a multiple of VEC here
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    const int w = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < KPW; ++j) ko[j] = __ldg(ktab + k0 + w * KPW + j);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < KPW; ++j) {
      const int k = w * KPW + j;
      float* row = sm + (k >> 2) * CH + 512 + (k & 3) * 128;
#pragma unroll
      for (int h = 0; h < 128 / NPL; ++h) {
        if constexpr (VEC == 4) cp_async16(row + NPL * h + 4 * l, g + (ro[h] + ko[j]), rv[h] && k0 + k < K);
        else cp_async8(row + NPL * h + 2 * l, g + (ro[h] + ko[j]), rv[h] && k0 + k < K);
      }
    }
  }
};

// B along N by shifted 16-byte vectors (mode 12, N = 256 form): B's N runs are contiguous but
// start at any 4-byte offset, so each run is copied as the aligned 16-byte blocks that cover it
// (tc_api.cpp nshift_tables: per tile block of 128 columns, run j gets ceil((L + 6) / 4) slots)
// into a [k][n] staging of 256 floats per k that spans the hi and lo halves of its K chunk. The
// blocks of K index k start at the run's aligned offset plus rscat_B[k] rounded down to 4, so
// column n sits at a per-column staging word plus the per-k shift rscat_B[k] mod 4; the
// converter warps pick the values out and write the K-major hi and lo rows over the staging.
template <typename IDX, int CH>
struct GatherSNV {
  static constexpr int KPW = BK / kPW;               // k rows per warp (8)
  static constexpr int NS = 64;                      // slots per tile block (tc_api.cpp)
  int2 ent[2];                                       // slots lane, lane + 32
  IDX ko[KPW];
  __device__ __forceinline__ void init_tab(const int* __restrict__ tab, int tn, int l) {
    const int2* t = reinterpret_cast<const int2*>(tab) + (size_t)tn * NS;
    ent[0] = t[l];
    ent[1] = t[l + 32];
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
    const int w = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < KPW; ++j) ko[j] = __ldg(ktab + k0 + w * KPW + j);
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < KPW; ++j) {
      const int k = w * KPW + j;
      float* row = sm + (k >> 2) * CH + (k & 3) * 256;
      const bool kin = k0 + k < K;
      const int kk = (int)ko[j];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        // block i of its run holds words [4 i, 4 i + 4) of the run shifted by c + (k mod 4):
        // copied when they overlap the run's L words (d = c + shift - 4 i)
        const int d = (ent[h].y & 0xFFF) - 2048 + (kk & 3), L = ent[h].y >> 12;
        if (d < 4 && d + L > 0) cp_async16(row + 4 * (l + 32 * h), g + (ent[h].x + (kk & ~3)), kin);
      }
    }
  }
};

// operand gather modes: 0 row-mapped elements, 1 K-run elements, 2 K vectors, 3 row vectors,
// 5 K pairs, 6 row pairs (A), 7 K-run elements one row per instruction, 8 rows one k per
// instruction
template <typename IDX, int MODE, int CH = kChunk, int ROWS = 128> struct GatherSel;
template <typename IDX, int CH, int R> struct GatherSel<IDX, 0, CH, R> { using type = Gather<IDX, false, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 1, CH, R> { using type = Gather<IDX, true, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 2, CH, R> { using type = GatherVK<IDX, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 3, CH, R> { using type = GatherVM<IDX>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 5, CH, R> { using type = GatherP2K<IDX, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 6, CH, R> { using type = GatherP2M<IDX>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 7, CH, R> { using type = GatherK32<IDX, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 8, CH, R> { using type = GatherR32<IDX, CH, R>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 10, CH, R> { using type = GatherVN<IDX, CH, 4>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 11, CH, R> { using type = GatherVN<IDX, CH, 2>; };
template <typename IDX, int CH, int R> struct GatherSel<IDX, 12, CH, R> { using type = GatherSNV<IDX, CH>; };

#ifdef TC_UMMA_PROF
// measurement build: per-role cycles spent in each barrier wait, printed by CTA 0 at exit
#define PWAIT(slot, stmt) { const long long t0_ = clock64(); stmt; prof[slot] += clock64() - t0_; }
#else
#define PWAIT(slot, stmt) stmt
#endif

__device__ __forceinline__ void epi_sync() {   // the four epilogue warps only
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
}

// Read-modify-write of one 32 x 32 block of C (32 rows of this warp, 32 columns) when C's unit
// stride runs along N: the block is staged transposed in shared memory (stg, written by the
// caller as [row][col], pitch 33), so each warp load / store covers 32 consecutive columns of
// one row instead of 32 rows. Out of line, so its registers stay out of the kernel's loops.
template <typename IDX>
__device__ __noinline__ void rmw_block_transposed(const float* stg, float* C, IDX rc, IDX col,
                                                  int mrow0, int M, bool cin, int piece,
                                                  double alpha, double beta, int lane) {
  float old[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const IDX rr = __shfl_sync(0xffffffffu, rc, r);
    old[r] = (cin && mrow0 + r < M) ? C[rr + col] : 0.f;
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const IDX rr = __shfl_sync(0xffffffffu, rc, r);
    double out = alpha * static_cast<double>(stg[r * 33 + lane]);
    out = piece > 0 ? out + static_cast<double>(old[r]) : fma(beta, static_cast<double>(old[r]), out);
    if (cin && mrow0 + r < M) C[rr + col] = static_cast<float>(out);
  }
}

// Stream-K fix-up of a later piece (piece > 0): the block's alpha * acc is added into C at L2
// with red.global.add.f32, no read of C (the flags still fix the order of the pieces, and the
// piece's fence before publishing waits for the reductions), through the same transpose.
// TC_UMMA_RED=0 (build flag): load-add-store instead (rmw_block_transposed).
#ifndef TC_UMMA_RED
#define TC_UMMA_RED 1
#endif
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
template <typename IDX>
__device__ __noinline__ void red_block_transposed(const float* stg, float* C, IDX rc, IDX col,
                                                  int mrow0, int M, bool cin, double alpha,
                                                  int lane) {
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const IDX rr = __shfl_sync(0xffffffffu, rc, r);
    if (cin && mrow0 + r < M)
      red_add_f32(C + (rr + col), static_cast<float>(alpha * static_cast<double>(stg[r * 33 + lane])));
  }
}

// Write-only counterpart (TC_UMMA_WT=1: measurement switch): alpha * block through the same
// transpose, one 128-byte row segment per warp store.
#ifndef TC_UMMA_WT
#define TC_UMMA_WT 0
#endif
template <typename IDX>
__device__ __noinline__ void store_block_transposed(const float* stg, float* C, IDX rc, IDX col,
                                                    int mrow0, int M, bool cin, double alpha,
                                                    int lane) {
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const IDX rr = __shfl_sync(0xffffffffu, rc, r);
    if (cin && mrow0 + r < M)
      C[rr + col] = static_cast<float>(alpha * static_cast<double>(stg[r * 33 + lane]));
  }
}

// cluster (CTA pair) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n"
               ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" :: "r"(r) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\nWAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITC_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mma_tf32_ta_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                                 uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               :: "r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {   // to both CTAs' barrier
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster"
               ".b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

template <typename IDX, int A_MODE, int B_MODE>
__global__ void __launch_bounds__(kThreads, 1)
tc_umma_f32_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                   const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                   const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                   const IDX* __restrict__ rC, const IDX* __restrict__ cC, int M, int N, int K,
                   int tiles_m, int tiles_n, double alpha, double beta, Sched sched,
                   int* __restrict__ flags, bool c_lanes_n, const int* __restrict__ bsh_p,
                   const int* __restrict__ bsh_c) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kChA = chunk_stride<128 * 4, A_MODE>();
  constexpr int kChB = chunk_stride<kChunkB - 16, B_MODE>();
  float* stage0 = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * kStage * sizeof(float));
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tfull = empty + STAGES;    // [kChunkBufs]
  uint64_t* tempty = tfull + kChunkBufs;
  uint64_t* aempty = tempty + kChunkBufs;   // [kASlots] (A in TMEM)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kASlots);
  float* epi_stage = reinterpret_cast<float*>(smem_raw + kEpiOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef TC_UMMA_PROF
  long long prof[6] = {0, 0, 0, 0, 0, 0};
  const long long tstart = clock64();
#endif
  const uint32_t crank = kPair ? cluster_rank() : 0;   // 0: the pair's leader (issues the MMAs)
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kPW * 32);
      mbar_init(&conv[s], (kPair ? 2 : 1) * kCW);   // one arrival per converter warp
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < kChunkBufs; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (kPair ? 2 : 1) * 128);
    }
    for (int a = 0; a < kASlots; ++a) mbar_init(&aempty[a], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kMmaW) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n"
                   :: "r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                   :: "r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if constexpr (kPair) cluster_sync_all();   // barriers of both CTAs initialised, TMEM allocated
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // every role walks the same work items: whole tiles, then this CTA's stream-K pieces
  // (sched.cuh); a piece is the K-step range [kb, ke) of one tile
  WorkIter wi;
  wi.init(sched, kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x);   // pair: one unit per cluster
  int tile, kb, ke;
  bool sk;

  if (warp < kPW) {
    // ---------------------------------- producers ----------------------------------
    typename GatherSel<IDX, A_MODE, kChA>::type ga;
    typename GatherSel<IDX, B_MODE, kChB, kRowsB>::type gb;
    uint32_t it = 0;
    // K offsets depend on the K step only: those of the next step are fetched while this one's
    // copies are in flight, so the table reads stay off the producer's critical path
    int kpre = 0;
    ga.load_k(cA, 0, lane);
    gb.load_k(rB, 0, lane);
    while (wi.next(tile, kb, ke, sk)) {
      int tm, tn;
      tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
      ga.init(rA, tm * kTM + BM * (int)crank, M, warp, lane);
      if constexpr (B_MODE == 12) gb.init_tab(bsh_p, tn, lane);
      else gb.init(cB, tn * BN + kRowsB * (int)crank, N, warp, lane);
      if (kpre != kb) {
        ga.load_k(cA, kb * BK, lane);
        gb.load_k(rB, kb * BK, lane);
      }
      for (int kt = kb; kt < ke; ++kt, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) PWAIT(0, mbar_wait(&empty[s], ((it / STAGES) - 1) & 1));
        float* st = stage0 + s * kStage;
        ga.issue(st, A, kt * BK, K, warp, lane);
        gb.issue(st + kOffBh, B, kt * BK, K, warp, lane);
        mbar_cp_async_arrive(&full[s]);
        kpre = kt + 1 < ke ? kt + 1 : 0;
        ga.load_k(cA, kpre * BK, lane);
        gb.load_k(rB, kpre * BK, lane);
      }
    }
    cp_async_wait_all();
  } else if (warp < kEpi0) {
    // ---------------------------------- converters ---------------------------------
    const int t = threadIdx.x - kConv0 * 32;
    uint32_t it = 0;
    while (wi.next(tile, kb, ke, sk)) {
      int cv = 0;   // mode 12: this thread's column's staging word (before the per-k shift)
      if constexpr (B_MODE == 12) {
        int tm, tn;
        tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
        cv = __ldg(bsh_c + tn * BN + t);
      }
      for (int kt = kb; kt < ke; ++kt, ++it) {
        const int s = it % STAGES;
        int kq = 0;   // mode 12: this lane's k (= lane) offset of the step, for the shifts
        if constexpr (B_MODE == 12) kq = kt * BK + lane < K ? (int)__ldg(rB + kt * BK + lane) : 0;
        PWAIT(1, mbar_wait(&full[s], (it / STAGES) & 1));
        float* st = stage0 + s * kStage;
        if constexpr (kN256 && B_MODE == 12) {
          // B from the shifted staging: column t's value of k sits at its run's slots + the
          // run's shift for k, ((cscat_B[s] + rscat_B[k]) mod 4); shifts of the 32 k as two
          // ballot masks
          static_assert(kCW == 4, "one converter thread per B row");
          const uint32_t m0 = __ballot_sync(0xffffffffu, kq & 1), m1 = __ballot_sync(0xffffffffu, kq & 2);
          const float* sb = st + kOffBh + cv;
          float v[BK];
#pragma unroll
          for (int k = 0; k < BK; ++k) {
            const int sh = (int)((m0 >> k) & 1u) | (int)(((m1 >> k) & 1u) << 1);   // warp-uniform
            v[k] = sb[(k >> 2) * kChB + (k & 3) * 256 + sh];
          }
          asm volatile("bar.sync 3, %0;\n" ::"n"(kCW * 32) : "memory");   // converters only
#pragma unroll
          for (int c = 0; c < BK / 4; ++c) {
            const float4 x = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            float4* hi = reinterpret_cast<float4*>(st + kOffBh + c * kChB) + t;
            *hi = x;
            hi[128] = make_float4(lo_round(x.x - tf32_trunc(x.x)), lo_round(x.y - tf32_trunc(x.y)),
                                  lo_round(x.z - tf32_trunc(x.z)), lo_round(x.w - tf32_trunc(x.w)));
          }
        } else if constexpr (kN256 && (B_MODE == 10 || B_MODE == 11)) {
          // B from the [k][n] staging in the lo halves: this thread's row n, all 32 K values
          // into registers, then (once every converter thread has read) the hi rows and the lo
          // rows over the staging
          static_assert(kCW == 4, "one converter thread per B row");
          float v[BK];
#pragma unroll
          for (int c = 0; c < BK / 4; ++c)
#pragma unroll
            for (int j = 0; j < 4; ++j) v[4 * c + j] = st[kOffBh + c * kChB + 512 + j * 128 + t];
          asm volatile("bar.sync 3, %0;\n" ::"n"(kCW * 32) : "memory");   // converters only
#pragma unroll
          for (int c = 0; c < BK / 4; ++c) {
            const float4 x = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
            float4* hi = reinterpret_cast<float4*>(st + kOffBh + c * kChB) + t;
            *hi = x;
            hi[128] = make_float4(lo_round(x.x - tf32_trunc(x.x)), lo_round(x.y - tf32_trunc(x.y)),
                                  lo_round(x.z - tf32_trunc(x.z)), lo_round(x.w - tf32_trunc(x.w)));
          }
        } else if constexpr (kN256) {
          // B: lo rows next to the hi rows of every K chunk
#pragma unroll
          for (int i = t; i < (BK / 4) * 128; i += kCW * 32) {
            float4* hi = reinterpret_cast<float4*>(st + kOffBh + (i >> 7) * kChB) + (i & 127);
            const float4 x = *hi;
            float4 h;
            h.x = tf32_trunc(x.x); h.y = tf32_trunc(x.y); h.z = tf32_trunc(x.z); h.w = tf32_trunc(x.w);
            hi[128] = make_float4(lo_round(x.x - h.x), lo_round(x.y - h.y), lo_round(x.z - h.z),
                                  lo_round(x.w - h.w));
          }
        } else {
#pragma unroll
        for (int op = kTmemA ? 1 : 0; op < 2; ++op) {   // A (in smem), then B: hi, lo buffers
          float4* hi = reinterpret_cast<float4*>(st + (op ? kOffBh : 0));
          float4* lo = reinterpret_cast<float4*>(st + (op ? kOffBl : kOffAl));
#pragma unroll
          for (int i = t; i < (op ? kTileB : kTile) / 4; i += kCW * 32) {
            const float4 x = hi[i];
            float4 h;
#if TC_UMMA_HI_TRUNC
            // hi stays the raw fp32 value: the tensor core reads only its tf32 bits (truncation),
            // so hi = trunc(x) and only lo = x - trunc(x) is written
            h.x = tf32_trunc(x.x); h.y = tf32_trunc(x.y); h.z = tf32_trunc(x.z); h.w = tf32_trunc(x.w);
#else
            h.x = tf32_rna(x.x); h.y = tf32_rna(x.y); h.z = tf32_rna(x.z); h.w = tf32_rna(x.w);
            hi[i] = h;
#endif
            // lo rounded to tf32 as well: the tensor core would otherwise truncate its low
            // mantissa bits, a bias that grows with K
            lo[i] = make_float4(lo_round(x.x - h.x), lo_round(x.y - h.y), lo_round(x.z - h.z),
                                lo_round(x.w - h.w));
          }
        }
        }
        if constexpr (kTmemA) {
          // A to tensor memory: this thread's row (TMEM lane 32 q + lane), 32 K values
          const int q = (warp - kConv0) & 3;
          constexpr int KC = BK * 4 / kCW;           // K columns per converter warp (32 or 16)
          const int kc0 = ((warp - kConv0) >> 2) * KC;
          const int row = 32 * q + lane;
          const uint32_t slot = it % kASlots;
          if (it >= kASlots) PWAIT(2, mbar_wait(&aempty[slot], ((it / kASlots) - 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          uint32_t h[KC], lo[KC];
#pragma unroll
          for (int c = 0; c < KC / 4; ++c) {
            const int k = kc0 + 4 * c;
            float4 x;
            if constexpr (A_MODE == 3 || A_MODE == 6) {   // [k][m] staging
              x = make_float4(st[k * BM + row], st[(k + 1) * BM + row], st[(k + 2) * BM + row],
                              st[(k + 3) * BM + row]);
            } else {
              x = *reinterpret_cast<const float4*>(st + tile_off<kChA>(row, k));
            }
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float hv = tf32_trunc(xs[e]);
              h[4 * c + e] = __float_as_uint(hv);
              lo[4 * c + e] = __float_as_uint(lo_round(xs[e] - hv));
            }
          }
          const uint32_t ta =
              tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(kACol + slot * 2 * BK + kc0);
          tmem_st_n(ta, h);
          tmem_st_n(ta + BK, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // visible to the MMA
        __syncwarp();   // every lane has fenced its writes; one arrival per warp
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_remote(&conv[s], 0);   // the leader's barrier
          else mbar_arrive(&conv[s]);
        }
      }
    }
  } else if (warp < kMmaW) {
    // ---------------------------------- epilogue -----------------------------------
    // TMEM columns: chunk accumulators at 0, 128, 256 (round robin), the item's running sum at 384
    const int q = warp - kEpi0;                // TMEM lane quarter of this warp
    const int row = 32 * q + lane;
    const uint32_t lanes = (uint32_t)(32 * q) << 16;
    uint32_t ch = 0;
#ifdef TC_UMMA_TRACE
    int ntr = 0, trm[4][4];
    unsigned long long trt[4][4];
#endif
    while (wi.next(tile, kb, ke, sk)) {
      int tm, tn;
      tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
      const int m = tm * kTM + BM * (int)crank + row;
      const bool min_ = m < M;
      const IDX rc = min_ ? rC[m] : 0;
      const int n0 = tn * BN;
      const int nchunks = (ke - kb + kChunkSteps - 1) / kChunkSteps;
      // stream-K piece order (sched.cuh): piece 0 writes alpha*acc + beta*C, piece j >= 1
      // waits for flag == j and adds alpha*acc; a piece that is not the last publishes j + 1
      const bool split = sk && !(kb == 0 && ke == sched.KT);
      int piece = 0;
      int* flag = nullptr;
      if (split) {
        const int s_local = tile - sched.D;
        const long long g_first = (long long)s_local * sched.KT;
        const int owner = (int)(((g_first + 1) * sched.P_sk + sched.I - 1) / sched.I) - 1;
        piece = (kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x) - owner;
        flag = flags + s_local;
      }
      const bool read_c = piece > 0 || beta != 0.0;
      // C's column offsets for the tile, one per lane and 32-column group, fetched now so the
      // final store does not start with a table round trip
      IDX colv[4];
#pragma unroll
      for (int g = 0; g < 4; ++g)
        colv[g] = n0 + 32 * g + lane < N ? __ldg(cC + n0 + 32 * g + lane) : 0;
#ifdef TC_UMMA_TRACE
      unsigned long long tr0, tr1 = 0, tr2 = 0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
#endif
      for (int c = 0; c < nchunks; ++c, ++ch) {
        const int cb = ch % kChunkBufs;
        const bool last = c == nchunks - 1;
        if (last && piece > 0) {
#ifdef TC_UMMA_TRACE
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
#endif
          // pair: each piece is published by both CTAs (two counts per piece)
          if (threadIdx.x == kEpi0 * 32)
          {
            if constexpr (kPair) wait_flag_ge(flag, sched.epoch, 2 * piece);
            else wait_flag(flag, (int)(sched.epoch | (unsigned)piece));
          }
          epi_sync();
#ifdef TC_UMMA_TRACE
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr2));
#endif
        }
        PWAIT(3, mbar_wait(&tfull[cb], (ch / kChunkBufs) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
        for (int c0 = 0; c0 < 4; ++c0) {
          uint32_t u[32];
          if constexpr (kN256) {
            // chunk = main (columns 0-127) + correction (128-255); the chunk accumulator is free
            // for the next chunk's MMAs as soon as its last columns are in registers
            {
              uint32_t v[32];
              tmem_ld32(tmem + lanes + (uint32_t)(32 * c0), u);
              tmem_ld32(tmem + lanes + (uint32_t)(BN + 32 * c0), v);
              asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
              for (int i = 0; i < 32; ++i)
                u[i] = __float_as_uint(__uint_as_float(u[i]) + __uint_as_float(v[i]));
            }
            if (c0 == 3) {
              asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
              if constexpr (kPair) mbar_arrive_remote(&tempty[cb], 0);
              else mbar_arrive(&tempty[cb]);
            }
            if (c > 0) {
              uint32_t t2[32];
              tmem_ld32(tmem + lanes + (uint32_t)(kSumCol + 32 * c0), t2);
              asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
              for (int i = 0; i < 32; ++i)
                u[i] = __float_as_uint(__uint_as_float(u[i]) + __uint_as_float(t2[i]));
            }
          } else {
          tmem_ld32(tmem + lanes + (uint32_t)(cb * BN + 32 * c0), u);
          if (c > 0) {
            uint32_t t2[32];
            tmem_ld32(tmem + lanes + (uint32_t)(kSumCol + 32 * c0), t2);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i)
              u[i] = __float_as_uint(__uint_as_float(u[i]) + __uint_as_float(t2[i]));
          } else {
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          }
          }
          if (!last) {
            tmem_st32(tmem + lanes + (uint32_t)(kSumCol + 32 * c0), u);
          } else {
            // final values of 32 columns: the column offsets (one coalesced load, shuffled
            // out), then all reads of C, then all stores, so the memory round trips overlap
            // instead of one dependent read per element
            const int nb = n0 + 32 * c0;
            const bool full = nb + 32 <= N;
            const IDX col = c0 == 0 ? colv[0] : c0 == 1 ? colv[1] : c0 == 2 ? colv[2] : colv[3];
            // (no branch on the row: the shuffles need the whole warp)
            if (read_c && c_lanes_n) {
              float* stg = epi_stage + q * 32 * 33;
#pragma unroll
              for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = __uint_as_float(u[i]);
              __syncwarp();
              if (TC_UMMA_RED && piece > 0)
                red_block_transposed<IDX>(stg, C, rc, col, m - lane, M, nb + lane < N, alpha, lane);
              else
                rmw_block_transposed<IDX>(stg, C, rc, col, m - lane, M, nb + lane < N, piece,
                                          alpha, beta, lane);
              __syncwarp();
            } else if (TC_UMMA_WT && !read_c && c_lanes_n) {
              float* stg = epi_stage + q * 32 * 33;
#pragma unroll
              for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = __uint_as_float(u[i]);
              __syncwarp();
              store_block_transposed<IDX>(stg, C, rc, col, m - lane, M, nb + lane < N, alpha, lane);
              __syncwarp();
            } else if (TC_UMMA_RED && piece > 0) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const IDX o = __shfl_sync(0xffffffffu, col, i);
                if (min_ && (full || nb + i < N))
                  red_add_f32(C + (rc + o),
                              static_cast<float>(alpha * static_cast<double>(__uint_as_float(u[i]))));
              }
            } else if (read_c) {
              float old[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const IDX o = __shfl_sync(0xffffffffu, col, i);
                old[i] = (min_ && (full || nb + i < N)) ? C[rc + o] : 0.f;
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const IDX o = __shfl_sync(0xffffffffu, col, i);
                double out = alpha * static_cast<double>(__uint_as_float(u[i]));
                out = piece > 0 ? out + static_cast<double>(old[i])
                                : fma(beta, static_cast<double>(old[i]), out);
                if (min_ && (full || nb + i < N)) C[rc + o] = static_cast<float>(out);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const IDX o = __shfl_sync(0xffffffffu, col, i);
                if (min_ && (full || nb + i < N))
                  C[rc + o] = static_cast<float>(alpha * static_cast<double>(__uint_as_float(u[i])));
              }
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        if constexpr (kPair) mbar_arrive_remote(&tempty[cb], 0);   // chunk cb is free now
        else if constexpr (!kN256) mbar_arrive(&tempty[cb]);
      }
      if (split) {
        // publish this piece (epoch-tagged: nothing is reset for the next launch)
        epi_sync();
        if (threadIdx.x == kEpi0 * 32) {
          __threadfence();
          if constexpr (kPair) {
            count_flag(flag, sched.epoch);   // one count per CTA of the pair
          } else if (ke < sched.KT) {
            st_release(flag, (int)(sched.epoch | (unsigned)(piece + 1)));
          }
        }
      }
#ifdef TC_UMMA_TRACE
      if (ntr < 4) {
        unsigned long long tr3;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr3));
        trm[ntr][0] = tile; trm[ntr][1] = kb; trm[ntr][2] = ke; trm[ntr][3] = piece;
        trt[ntr][0] = tr0; trt[ntr][1] = tr1; trt[ntr][2] = tr2; trt[ntr][3] = tr3;
        ++ntr;
      }
#endif
    }
#ifdef TC_UMMA_TRACE
    if (threadIdx.x == kEpi0 * 32)
      for (int i = 0; i < ntr; ++i)
        printf("TR cta %d tile %d kb %d ke %d piece %d start %llu wait0 %llu wait1 %llu end %llu\n",
               (int)blockIdx.x, trm[i][0], trm[i][1], trm[i][2], trm[i][3], trt[i][0], trt[i][1],
               trt[i][2], trt[i][3]);
#endif
  } else {
    // ---------------------------------- MMA issuer ---------------------------------
    const uint32_t idesc256 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(2 * BN >> 3) << 17) |
                              ((uint32_t)(BM >> 4) << 24);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(kTM >> 4) << 24);   // pair: M = 256 across the two CTAs
    uint32_t it = 0, ch = 0;
    while ((!kPair || crank == 0) && wi.next(tile, kb, ke, sk)) {
      uint32_t d = 0;
      for (int kt = kb; kt < ke; ++kt, ++it) {
        const int j0 = (kt - kb) % kChunkSteps;
        const bool chunk_start = j0 == 0;
        const bool chunk_end = j0 == kChunkSteps - 1 || kt == ke - 1;
        if (chunk_start) {
          const int cb = ch % kChunkBufs;
          if (ch >= kChunkBufs) {
            if constexpr (kPair) { PWAIT(4, mbar_wait_cluster(&tempty[cb], ((ch / kChunkBufs) - 1) & 1)); }
            else { PWAIT(4, mbar_wait(&tempty[cb], ((ch / kChunkBufs) - 1) & 1)); }
          }
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          d = tmem + (uint32_t)(cb * kChunkCols);
        }
        const int s = it % STAGES;
        if constexpr (kPair) { PWAIT(5, mbar_wait_cluster(&conv[s], (it / STAGES) & 1)); }
        else { PWAIT(5, mbar_wait(&conv[s], (it / STAGES) & 1)); }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const float* st = stage0 + s * kStage;
          const float* bh = st + kOffBh;
          const float* bl = st + kOffBl;
          if constexpr (kPair) {
            const uint32_t slot = it % kASlots;
            const uint32_t ah = tmem + (uint32_t)(kACol + slot * 2 * BK), al = ah + BK;
#pragma unroll
            for (int j = 0; j < BK / 8; ++j) {
              const uint32_t acc0 = (!chunk_start || j > 0) ? 1u : 0u;
              const uint64_t dbh = make_desc<kChB>(bh, j), dbl = make_desc<kChB>(bl, j);
              mma_tf32_ta_pair(d, ah + 8 * j, dbh, idesc, acc0);
              mma_tf32_ta_pair(d, ah + 8 * j, dbl, idesc, 1u);
              mma_tf32_ta_pair(d, al + 8 * j, dbh, idesc, 1u);
            }
            mma_commit_pair(&aempty[slot]);            // both CTAs' A slots are free
          } else if constexpr (kN256) {
            const uint32_t slot = it % kASlots;
            const uint32_t ah = tmem + (uint32_t)(kACol + slot * 2 * BK), al = ah + BK;
#pragma unroll
            for (int j = 0; j < BK / 8; ++j) {
              const uint32_t acc0 = (!chunk_start || j > 0) ? 1u : 0u;
              const uint64_t db = make_desc<kChB>(bh, j);
              mma_tf32_ta(d, ah + 8 * j, db, idesc256, acc0);      // [Ahi.Bhi | Ahi.Blo]
              mma_tf32_ta(d + BN, al + 8 * j, db, idesc, 1u);      // + Alo.Bhi
            }
            mma_commit(&aempty[slot]);                 // A slot free once these complete
          } else if constexpr (kTmemA) {
            const uint32_t slot = it % kASlots;
            const uint32_t ah = tmem + (uint32_t)(kACol + slot * 2 * BK), al = ah + BK;
#pragma unroll
            for (int j = 0; j < BK / 8; ++j) {
              const uint32_t acc0 = (!chunk_start || j > 0) ? 1u : 0u;
              mma_tf32_ta(d, ah + 8 * j, make_desc<kChB>(bh, j), idesc, acc0);
              mma_tf32_ta(d, ah + 8 * j, make_desc<kChB>(bl, j), idesc, 1u);
              mma_tf32_ta(d, al + 8 * j, make_desc<kChB>(bh, j), idesc, 1u);
            }
            mma_commit(&aempty[slot]);                 // A slot free once these complete
          } else {
            const float* ah = st;
            const float* al = st + kOffAl;
#pragma unroll
            for (int j = 0; j < BK / 8; ++j) {
              const uint32_t acc0 = (!chunk_start || j > 0) ? 1u : 0u;
              mma_tf32(d, make_desc<kChA>(ah, j), make_desc<kChB>(bh, j), idesc, acc0);
              mma_tf32(d, make_desc<kChA>(ah, j), make_desc<kChB>(bl, j), idesc, 1u);
              mma_tf32(d, make_desc<kChA>(al, j), make_desc<kChB>(bh, j), idesc, 1u);
            }
          }
          if constexpr (kPair) {
            mma_commit_pair(&empty[s]);
            if (chunk_end) mma_commit_pair(&tfull[ch % kChunkBufs]);
          } else {
            mma_commit(&empty[s]);                     // stage s is free once these complete
            if (chunk_end) mma_commit(&tfull[ch % kChunkBufs]);   // the chunk is complete
          }
        }
        __syncwarp();
        if (chunk_end) ++ch;
      }
    }
  }

#ifdef TC_UMMA_PROF
  if (blockIdx.x == 0 && lane == 0)
    printf("PROF warp %d total %lld empty %lld full %lld aempty %lld tfull %lld tempty %lld conv %lld\n",
           warp, clock64() - tstart, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5]);
#endif
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if constexpr (kPair) cluster_sync_all();   // neither CTA frees TMEM the pair still uses
  else __syncthreads();
  if (warp == kMmaW) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" :: "r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tmem));
  }
}

template <typename IDX, int A_MODE, int B_MODE>
static int launch_dir(const LaunchArgs& a, cudaStream_t s) {
  constexpr int smem = kSmemBytes;
  auto kern = tc_umma_f32_kernel<IDX, A_MODE, B_MODE>;
  static std::atomic<int> attr[kMaxDevices];
  if (!ensure_dyn_smem(kern, smem, attr)) return -1;
  const int tiles_m = (a.M + kTM - 1) / kTM, tiles_n = (a.N + BN - 1) / BN;
  const int KT = (a.K + BK - 1) / BK;
  const int T = tiles_m * tiles_n;
  const int units = kPair ? a.num_sms / 2 : a.num_sms;   // schedule units: CTAs or CTA pairs
  // stream-K only when the partial wave is < 70% full: split pieces cost this kernel more than
  // the DMMA one (cfg4 fp32: a 74-86% partial wave ran 8-13% faster whole, a < 30% one 10-20%
  // faster split; profiles/r01/ab_umma_sk.txt). TC_UMMA_SK=0 turns the tail off.
  const char* pe = getenv("TC_UMMA_SK");
  const bool sk = a.stream_k && !(pe && !strcmp(pe, "0"));
  const char* pp = getenv("TC_UMMA_DPPCT");   // measurement override of the 70% threshold
  // stream-K pieces of at least min(KT, 16) K steps (and 8): this kernel's fix-up links are
  // expensive, so few, longer pieces win on small problems (1024^3: 0.58 -> 0.99 of SGEMM,
  // 512^3 0.34 -> 0.46; profiles/r01/ab_min_sk.txt)
  const int min_sk = KT < 8 ? 8 : (KT > 16 ? 16 : KT);
  Sched sc = make_sched(T, KT, units, sk, pp ? atoi(pp) : 70, min_sk);
  if (sc.P_sk > 0 && (sc.T - sc.D) > a.flags_cap) sc = make_sched(T, KT, units, false);
  sc.wave_sync = 0;
  sc.epoch = a.flag_epoch;
  const int nunits = sc.D > 0 ? (sc.D < sc.P ? sc.D : sc.P) : sc.P_sk;
  const float* pA = static_cast<const float*>(a.A);
  const float* pB = static_cast<const float*>(a.B);
  float* pC = static_cast<float*>(a.C);
  const IDX *trA = static_cast<const IDX*>(a.rA), *tcA = static_cast<const IDX*>(a.cA);
  const IDX *trB = static_cast<const IDX*>(a.rB), *tcB = static_cast<const IDX*>(a.cB);
  const IDX *trC = static_cast<const IDX*>(a.rC), *tcC = static_cast<const IDX*>(a.cC);
  if constexpr (kPair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * nunits);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeClusterDimension;
    attr1[0].val.clusterDim.x = 2;
    attr1[0].val.clusterDim.y = 1;
    attr1[0].val.clusterDim.z = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, pA, pB, pC, trA, tcA, trB, tcB, trC, tcC, a.M, a.N, a.K,
                           tiles_m, tiles_n, a.alpha, a.beta, sc, a.flags, a.c_lanes_n,
                           a.bsh_p, a.bsh_c) != cudaSuccess)
      return -1;
  } else {
    kern<<<nunits, kThreads, smem, s>>>(pA, pB, pC, trA, tcA, trB, tcB, trC, tcC, a.M, a.N, a.K,
                                        tiles_m, tiles_n, a.alpha, a.beta, sc, a.flags,
                                        a.c_lanes_n, a.bsh_p, a.bsh_c);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace TC_UMMA_NS

// fp32 through the tensor cores (3xTF32). Applies to int32-offset fp32 contractions with
// K >= 1. The gather of each operand follows its leading direction (plan.cpp: A is read along M
// when a_vec_m, B along K when b_vec_k) and uses 16-byte vectors when the plan proved them all
// contiguous and aligned (a_vec_all / b_vec_all); an N-contiguous B is always element-gathered
// (its vectors would not be contiguous in the K-major MMA layout).
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int TC_UMMA_LAUNCH(const LaunchArgs& a, cudaStream_t stream) {
  if (!a.f32 || a.idx64 || a.K < 1) return 0;
  using namespace TC_UMMA_NS;
  // 8-byte pair gathers where the operand's pairs (not all its vectors) are contiguous and
  // aligned (TC_UMMA_PAIRS=0: off); element gathers one line per instruction (modes 7 / 8;
  // TC_UMMA_MAP=0: the 4 x 8 / 8 x 4 mappings, modes 1 / 0). Measurement switches, read per call.
  const char* pe2 = getenv("TC_UMMA_PAIRS");
  const char* pm = getenv("TC_UMMA_MAP");
  const bool pairs = !kPair && !(pe2 && !strcmp(pe2, "0"));
  // TC_UMMA_MAP (measurement; default "kr"): 'k' = K gathers one row per instruction (both
  // operands), 'r' = A's row gathers one k per instruction, 'b' = B's as well. Measured on cfg4
  // (profiles/r02/ab_umma_lines.txt): K gathers +10-32% where the K traversal interleaves
  // dimensions (cfg4_05, 06, 11), neutral elsewhere; A's row gathers +4-11% (cfg4_04, 07, 18);
  // B's row gathers -3..-9% on most cases whose B rows are contiguous (the 4-way bank conflicts of
  // 32 rows at one k in the K-major layout cost more than the lines they save), so off
  const bool mk = !kPair && (!pm || strchr(pm, 'k'));
  const bool mr = !kPair && (!pm || strchr(pm, 'r')), mb = !kPair && pm && strchr(pm, 'b');
  const bool a2 = pairs && a.a_vec2_all, b2 = pairs && a.b_vec2_all;
  const int a_row = mr ? 8 : 0, a_k = mk ? 7 : 1;   // element modes
  const int b_row = mb ? 8 : 0, b_k = mk ? 7 : 1;
#ifdef TC_UMMA_ELEM_ONLY
  // TC_UMMA_BN=0: B along N by elements even where its N vectors / pairs qualify (measurement)
  const char* pbn = getenv("TC_UMMA_BN");
  const bool bn = !(pbn && !strcmp(pbn, "0"));
  // TC_UMMA_AM=0: no 16-byte M vectors for A in this form (measurement)
  const char* pam = getenv("TC_UMMA_AM");
  const bool amv = !(pam && !strcmp(pam, "0"));
  // TC_UMMA_KV=1: 16-byte K vectors (mode 2) in this form too (measurement)
  const char* pkv = getenv("TC_UMMA_KV");
  const bool kv = pkv && !strcmp(pkv, "1");
  const int am = a.a_vec_m ? (amv && a.a_vec_all ? 3 : (a2 ? 6 : a_row))
                           : (kv && a.a_vec_all ? 2 : (a2 ? 5 : a_k));
  // B's shifted N vectors (mode 12) pay where A's gathers are element copies one k per
  // instruction (mode 8): there the producers bound the kernel and mode 12 halves B's copy
  // instructions (cfg4_07 +13%, cfg4_18 +10%); with cheaper A gathers the converters' extra work
  // (scalar staging reads, the hi rows rewritten) costs more than it saves (cfg4_02, 06, 14:
  // -3..-4%; profiles/r02/ab_umma_shift.txt). TC_UMMA_SHIFT=2 forces it wherever available.
  const bool shift = bn && (a.b_shift == 2 || (a.b_shift == 1 && am == 8));
  const int bm = a.b_vec_k ? (kv && a.b_vec_all ? 2 : (b2 ? 5 : b_k))
                           : (bn && a.b_vec_all ? 10 : (bn && b2 ? 11 : (shift ? 12 : b_row)));
  if (getenv("TC_UMMA_DEBUG")) fprintf(stderr, "tc_umma n256: A mode %d, B mode %d\n", am, bm);
  if constexpr (!kPair) {
    switch (am * 100 + bm) {
    case 0: return launch_dir<int, 0, 0>(a, stream);
    case 1: return launch_dir<int, 0, 1>(a, stream);
    case 5: return launch_dir<int, 0, 5>(a, stream);
    case 7: return launch_dir<int, 0, 7>(a, stream);
    case 8: return launch_dir<int, 0, 8>(a, stream);
    case 100: return launch_dir<int, 1, 0>(a, stream);
    case 101: return launch_dir<int, 1, 1>(a, stream);
    case 105: return launch_dir<int, 1, 5>(a, stream);
    case 107: return launch_dir<int, 1, 7>(a, stream);
    case 108: return launch_dir<int, 1, 8>(a, stream);
    case 500: return launch_dir<int, 5, 0>(a, stream);
    case 501: return launch_dir<int, 5, 1>(a, stream);
    case 505: return launch_dir<int, 5, 5>(a, stream);
    case 507: return launch_dir<int, 5, 7>(a, stream);
    case 508: return launch_dir<int, 5, 8>(a, stream);
    case 600: return launch_dir<int, 6, 0>(a, stream);
    case 601: return launch_dir<int, 6, 1>(a, stream);
    case 605: return launch_dir<int, 6, 5>(a, stream);
    case 607: return launch_dir<int, 6, 7>(a, stream);
    case 608: return launch_dir<int, 6, 8>(a, stream);
    case 700: return launch_dir<int, 7, 0>(a, stream);
    case 701: return launch_dir<int, 7, 1>(a, stream);
    case 705: return launch_dir<int, 7, 5>(a, stream);
    case 707: return launch_dir<int, 7, 7>(a, stream);
    case 708: return launch_dir<int, 7, 8>(a, stream);
    case 800: return launch_dir<int, 8, 0>(a, stream);
    case 801: return launch_dir<int, 8, 1>(a, stream);
    case 805: return launch_dir<int, 8, 5>(a, stream);
    case 807: return launch_dir<int, 8, 7>(a, stream);
    case 10: return launch_dir<int, 0, 10>(a, stream);
    case 11: return launch_dir<int, 0, 11>(a, stream);
    case 110: return launch_dir<int, 1, 10>(a, stream);
    case 111: return launch_dir<int, 1, 11>(a, stream);
    case 510: return launch_dir<int, 5, 10>(a, stream);
    case 511: return launch_dir<int, 5, 11>(a, stream);
    case 610: return launch_dir<int, 6, 10>(a, stream);
    case 611: return launch_dir<int, 6, 11>(a, stream);
    case 710: return launch_dir<int, 7, 10>(a, stream);
    case 711: return launch_dir<int, 7, 11>(a, stream);
    case 810: return launch_dir<int, 8, 10>(a, stream);
    case 811: return launch_dir<int, 8, 11>(a, stream);
    case 300: return launch_dir<int, 3, 0>(a, stream);
    case 301: return launch_dir<int, 3, 1>(a, stream);
    case 305: return launch_dir<int, 3, 5>(a, stream);
    case 307: return launch_dir<int, 3, 7>(a, stream);
    case 308: return launch_dir<int, 3, 8>(a, stream);
    case 310: return launch_dir<int, 3, 10>(a, stream);
    case 311: return launch_dir<int, 3, 11>(a, stream);
    case 2: return launch_dir<int, 0, 2>(a, stream);
    case 102: return launch_dir<int, 1, 2>(a, stream);
    case 200: return launch_dir<int, 2, 0>(a, stream);
    case 201: return launch_dir<int, 2, 1>(a, stream);
    case 202: return launch_dir<int, 2, 2>(a, stream);
    case 205: return launch_dir<int, 2, 5>(a, stream);
    case 207: return launch_dir<int, 2, 7>(a, stream);
    case 208: return launch_dir<int, 2, 8>(a, stream);
    case 210: return launch_dir<int, 2, 10>(a, stream);
    case 211: return launch_dir<int, 2, 11>(a, stream);
    case 302: return launch_dir<int, 3, 2>(a, stream);
    case 502: return launch_dir<int, 5, 2>(a, stream);
    case 602: return launch_dir<int, 6, 2>(a, stream);
    case 702: return launch_dir<int, 7, 2>(a, stream);
    case 802: return launch_dir<int, 8, 2>(a, stream);
    case 12: return launch_dir<int, 0, 12>(a, stream);
    case 112: return launch_dir<int, 1, 12>(a, stream);
    case 212: return launch_dir<int, 2, 12>(a, stream);
    case 312: return launch_dir<int, 3, 12>(a, stream);
    case 512: return launch_dir<int, 5, 12>(a, stream);
    case 612: return launch_dir<int, 6, 12>(a, stream);
    case 712: return launch_dir<int, 7, 12>(a, stream);
    case 812: return launch_dir<int, 8, 12>(a, stream);
    default: return launch_dir<int, 8, 8>(a, stream);
    }
  }
#else
  const int am = a.a_vec_m ? (a.a_vec_all ? 3 : (a2 ? 6 : a_row)) : (a.a_vec_all ? 2 : (a2 ? 5 : a_k));
  const int bm = a.b_vec_k ? (a.b_vec_all ? 2 : (b2 ? 5 : b_k)) : b_row;
  if constexpr (!kPair) {
    switch (am * 10 + bm) {
    case 0: return launch_dir<int, 0, 0>(a, stream);
    case 1: return launch_dir<int, 0, 1>(a, stream);
    case 2: return launch_dir<int, 0, 2>(a, stream);
    case 5: return launch_dir<int, 0, 5>(a, stream);
    case 7: return launch_dir<int, 0, 7>(a, stream);
    case 8: return launch_dir<int, 0, 8>(a, stream);
    case 10: return launch_dir<int, 1, 0>(a, stream);
    case 11: return launch_dir<int, 1, 1>(a, stream);
    case 12: return launch_dir<int, 1, 2>(a, stream);
    case 15: return launch_dir<int, 1, 5>(a, stream);
    case 17: return launch_dir<int, 1, 7>(a, stream);
    case 18: return launch_dir<int, 1, 8>(a, stream);
    case 20: return launch_dir<int, 2, 0>(a, stream);
    case 21: return launch_dir<int, 2, 1>(a, stream);
    case 22: return launch_dir<int, 2, 2>(a, stream);
    case 25: return launch_dir<int, 2, 5>(a, stream);
    case 27: return launch_dir<int, 2, 7>(a, stream);
    case 28: return launch_dir<int, 2, 8>(a, stream);
    case 30: return launch_dir<int, 3, 0>(a, stream);
    case 31: return launch_dir<int, 3, 1>(a, stream);
    case 32: return launch_dir<int, 3, 2>(a, stream);
    case 35: return launch_dir<int, 3, 5>(a, stream);
    case 37: return launch_dir<int, 3, 7>(a, stream);
    case 38: return launch_dir<int, 3, 8>(a, stream);
    case 50: return launch_dir<int, 5, 0>(a, stream);
    case 51: return launch_dir<int, 5, 1>(a, stream);
    case 52: return launch_dir<int, 5, 2>(a, stream);
    case 55: return launch_dir<int, 5, 5>(a, stream);
    case 57: return launch_dir<int, 5, 7>(a, stream);
    case 58: return launch_dir<int, 5, 8>(a, stream);
    case 60: return launch_dir<int, 6, 0>(a, stream);
    case 61: return launch_dir<int, 6, 1>(a, stream);
    case 62: return launch_dir<int, 6, 2>(a, stream);
    case 65: return launch_dir<int, 6, 5>(a, stream);
    case 67: return launch_dir<int, 6, 7>(a, stream);
    case 68: return launch_dir<int, 6, 8>(a, stream);
    case 70: return launch_dir<int, 7, 0>(a, stream);
    case 71: return launch_dir<int, 7, 1>(a, stream);
    case 72: return launch_dir<int, 7, 2>(a, stream);
    case 75: return launch_dir<int, 7, 5>(a, stream);
    case 77: return launch_dir<int, 7, 7>(a, stream);
    case 78: return launch_dir<int, 7, 8>(a, stream);
    case 80: return launch_dir<int, 8, 0>(a, stream);
    case 81: return launch_dir<int, 8, 1>(a, stream);
    case 82: return launch_dir<int, 8, 2>(a, stream);
    case 85: return launch_dir<int, 8, 5>(a, stream);
    case 87: return launch_dir<int, 8, 7>(a, stream);
    default: return launch_dir<int, 8, 8>(a, stream);
    }
  }
  switch (am * 10 + bm) {
    case 0: return launch_dir<int, 0, 0>(a, stream);
    case 1: return launch_dir<int, 0, 1>(a, stream);
    case 2: return launch_dir<int, 0, 2>(a, stream);
    case 10: return launch_dir<int, 1, 0>(a, stream);
    case 11: return launch_dir<int, 1, 1>(a, stream);
    case 12: return launch_dir<int, 1, 2>(a, stream);
    case 20: return launch_dir<int, 2, 0>(a, stream);
    case 21: return launch_dir<int, 2, 1>(a, stream);
    case 22: return launch_dir<int, 2, 2>(a, stream);
    case 30: return launch_dir<int, 3, 0>(a, stream);
    case 31: return launch_dir<int, 3, 1>(a, stream);
    default: return launch_dir<int, 3, 2>(a, stream);
  }
#endif
}

}  // namespace tcb
