// fp32 contraction on the 5th-generation tensor cores (sm_100a tcgen05, kind::tf32) with the
// 3xTF32 split: every fp32 operand x is split into hi = tf32(x) and lo = x - hi, and
// A.B = Ahi.Bhi + Ahi.Blo + Alo.Bhi (the Alo.Blo term, ~2^-22 relative, is dropped), accumulated
// in fp32 in tensor memory. The error stays at fp32 level (plain TF32 would be ~1e-3); the
// normwise bound 1e-5 of BASELINE north_star is checked by the parity tests.
//
// The paper's method is unchanged: the tiles are gathered from the tensors' strides through the
// scatter vectors -- here straight into the tensor cores' canonical
// shared-memory layout -- and C is written through its scatter vectors with alpha / beta
// (P:605-616). One CTA per SM walks 128 x 128 tiles of C:
//   warps 0-3   producers: cp.async element gathers of A and B (128 x 32 each per K step) into
//               the stage's hi buffers in the K-major canonical layout; each warp instruction
//               fills one 128-byte core matrix (8 rows x 4 K), so shared-memory writes are
//               conflict free and global reads come in 32-byte runs from an M/N-contiguous
//               operand (8 rows) or 16-byte runs from a K-contiguous one (4 K)
//   warps 4-7   converters: split each staged element into hi (in place) and lo (second buffer)
//   warps 8-11  epilogue: tcgen05.ld of the accumulator (warp w reads TMEM lanes 32 (w - 8)..),
//               one row of C per thread, alpha * acc + beta * C through rscat_C / cscat_C
//   warp 12     MMA issuer: one lane issues 3 x 4 tcgen05.mma (M = N = 128, K = 8) per K step and
//               commits them to the stage's `empty` barrier; two TMEM accumulators let the
//               epilogue of tile t overlap the MMAs of tile t + 1.
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"

namespace tcb {
namespace umma {

using namespace dev;

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int kThreads = 13 * 32;
constexpr int kTile = BM * BK;           // floats per operand tile (BM == BN)
constexpr int kStage = 4 * kTile;        // A hi, A lo, B hi, B lo
constexpr int GROUP_M = 2;
// The tensor core's fp32 accumulation drifts with the number of MMA steps it chains (3xTF32 at
// K = 513: 3.7e-6 normwise, growing with K), so the accumulator restarts every kChunkSteps K
// steps; the epilogue warps add the chunk into a running sum held in TMEM (rounded fp32 adds).
constexpr int kChunkSteps = 4;             // K steps of BK per chunk (K = 128)

__device__ __forceinline__ uint32_t tmem_u32_addr(const void* p) { return smem_u32(p); }

// Canonical SWIZZLE_NONE layouts (CUTLASS UMMA conventions, in floats):
//  K-major : core matrix = 8 rows x 4 K (16 B per row); row groups of 8 at 32 floats (SBO 128 B),
//            K chunks of 4 at 512 floats (LBO 2 KB); one K = 8 MMA step spans two K chunks
//  MN-major: core matrix = 8 K x 4 rows (16 B per K); row groups of 4 at 32 floats (SBO 128 B),
//            K groups of 8 at 1024 floats (LBO 4 KB); one MMA step is one K group
template <bool MN>
__device__ __forceinline__ int tile_off(int r, int k) {
  return MN ? (k >> 3) * 1024 + (r >> 2) * 32 + (k & 7) * 4 + (r & 3)
            : (k >> 2) * 512 + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}

template <bool MN>
__device__ __forceinline__ uint64_t make_desc(const float* base, int j) {   // MMA step j (K 8j..)
  const uint32_t addr = smem_u32(base + j * 1024);
  const uint32_t lbo = MN ? 4096 : 2048, sbo = 128;
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
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// Producer side of one operand X (A: rows = M, B: rows = N). MN: gathered along its rows.
// Warp w covers a quarter of the tile's core matrices; lane l is element (l & 3 | l >> 2) of
// each core matrix it copies.
template <typename IDX, bool MN>
struct Gather {
  static constexpr int NR = MN ? 8 : 4;    // row groups per warp (of 4 or 8 rows)
  static constexpr int NK = MN ? 4 : 8;    // K groups per stage (of 8 or 4)
  IDX ro[NR];
  uint32_t rv;
  IDX ko[NK];
  __device__ __forceinline__ void init(const IDX* __restrict__ rtab, int base, int extent, int w,
                                       int l) {
    rv = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int r = base + (MN ? 4 * (w * NR + i) + (l & 3) : 8 * (w * NR + i) + (l >> 2));
      ro[i] = rtab[r];                       // tables are padded past the extent
      rv |= (r < extent ? 1u : 0u) << i;
    }
  }
  __device__ __forceinline__ void load_k(const IDX* __restrict__ ktab, int k0, int l) {
#pragma unroll
    for (int j = 0; j < NK; ++j) ko[j] = __ldg(ktab + k0 + (MN ? 8 * j + (l >> 2) : 4 * j + (l & 3)));
  }
  __device__ __forceinline__ void issue(float* sm, const float* __restrict__ g, int k0, int K, int w,
                                        int l) {
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      const int kk = MN ? 8 * j + (l >> 2) : 4 * j + (l & 3);
      const bool kin = k0 + kk < K;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int r = MN ? 4 * (w * NR + i) + (l & 3) : 8 * (w * NR + i) + (l >> 2);
        cp_async4(sm + tile_off<MN>(r, kk), g + (ro[i] + ko[j]), kin && ((rv >> i) & 1u));
      }
    }
  }
};

template <typename IDX, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
tc_umma_f32_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                   const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                   const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                   const IDX* __restrict__ rC, const IDX* __restrict__ cC, int M, int N, int K,
                   int tiles_m, int tiles_n, double alpha, double beta) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  float* stage0 = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * kStage * sizeof(float));
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tfull = empty + STAGES;    // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 128);
      mbar_init(&conv[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                 :: "r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int T = tiles_m * tiles_n;
  const int KT = (K + BK - 1) / BK;

  if (warp < 4) {
    // ---------------------------------- producers ----------------------------------
    Gather<IDX, A_MN> ga;
    Gather<IDX, B_MN> gb;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
      int tm, tn;
      tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
      ga.init(rA, tm * BM, M, warp, lane);
      gb.init(cB, tn * BN, N, warp, lane);
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        ga.load_k(cA, kt * BK, lane);
        gb.load_k(rB, kt * BK, lane);
        float* st = stage0 + s * kStage;
        ga.issue(st, A, kt * BK, K, warp, lane);
        gb.issue(st + 2 * kTile, B, kt * BK, K, warp, lane);
        mbar_cp_async_arrive(&full[s]);
      }
    }
    cp_async_wait_all();
  } else if (warp < 8) {
    // ---------------------------------- converters ---------------------------------
    const int t = threadIdx.x - 128;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        float* st = stage0 + s * kStage;
#pragma unroll
        for (int op = 0; op < 2; ++op) {          // A, then B: hi buffer, lo buffer after it
          float4* hi = reinterpret_cast<float4*>(st + op * 2 * kTile);
          float4* lo = reinterpret_cast<float4*>(st + op * 2 * kTile + kTile);
#pragma unroll
          for (int i = t; i < kTile / 4; i += 128) {
            const float4 x = hi[i];
            float4 h;
            h.x = tf32_rna(x.x); h.y = tf32_rna(x.y); h.z = tf32_rna(x.z); h.w = tf32_rna(x.w);
            hi[i] = h;
            // lo rounded to tf32 as well: the tensor core would otherwise truncate its low
            // mantissa bits, a bias that grows with K
            lo[i] = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z),
                                tf32_rna(x.w - h.w));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // visible to the MMA
#ifdef TC_UMMA_DEBUG
        if (blockIdx.x == 0 && it == 0 && t == 0) {
          printf("A_MN=%d B_MN=%d K=%d M=%d N=%d\n", (int)A_MN, (int)B_MN, K, M, N);
          for (int i = 0; i < 8; ++i)
            printf(" Ahi[%d]=%f Alo=%g Bhi[%d]=%f Blo=%g\n", i, st[i], st[kTile + i], i,
                   st[2 * kTile + i], st[3 * kTile + i]);
          printf(" A(r=1,k=0)=%f A(r=0,k=1)=%f B(r=1,k=0)=%f B(r=0,k=1)=%f\n",
                 st[tile_off<A_MN>(1, 0)], st[tile_off<A_MN>(0, 1)],
                 st[2 * kTile + tile_off<B_MN>(1, 0)], st[2 * kTile + tile_off<B_MN>(0, 1)]);
        }
#endif
        mbar_arrive(&conv[s]);
      }
    }
  } else if (warp < 12) {
    // ---------------------------------- epilogue -----------------------------------
    // TMEM columns: chunk accumulators at 0 and 128 (alternating), the tile's running sum at 256
    const int q = warp - 8;                 // TMEM lane quarter of this warp
    const int row = 32 * q + lane;
    const uint32_t lanes = (uint32_t)(32 * q) << 16;
    const int nchunks = (KT + kChunkSteps - 1) / kChunkSteps;
    uint32_t ch = 0;
    for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
      int tm, tn;
      tile_coords<GROUP_M>(tile, tiles_m, tiles_n, &tm, &tn);
      const int m = tm * BM + row;
      const bool min_ = m < M;
      const IDX rc = min_ ? rC[m] : 0;
      const int n0 = tn * BN;
      for (int c = 0; c < nchunks; ++c, ++ch) {
        const int cb = ch & 1;
        mbar_wait(&tfull[cb], (ch >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const bool last = c == nchunks - 1;
#pragma unroll 1
        for (int c0 = 0; c0 < 4; ++c0) {
          uint32_t u[32];
          tmem_ld32(tmem + lanes + (uint32_t)(cb * BN + 32 * c0), u);
          if (c > 0) {
            uint32_t t2[32];
            tmem_ld32(tmem + lanes + (uint32_t)(2 * BN + 32 * c0), t2);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i)
              u[i] = __float_as_uint(__uint_as_float(u[i]) + __uint_as_float(t2[i]));
          } else {
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          }
          if (!last) {
            tmem_st32(tmem + lanes + (uint32_t)(2 * BN + 32 * c0), u);
          } else if (min_) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int n = n0 + 32 * c0 + i;
              if (n < N) {
                float* p = C + (rc + __ldg(cC + n));
                double out = alpha * static_cast<double>(__uint_as_float(u[i]));
                if (beta != 0.0) out = fma(beta, static_cast<double>(*p), out);
                *p = static_cast<float>(out);
              }
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(&tempty[cb]);           // chunk accumulator cb may be overwritten now
      }
    }
  } else {
    // ---------------------------------- MMA issuer ---------------------------------
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                           ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    uint32_t it = 0, ch = 0;
    for (int tile = blockIdx.x; tile < T; tile += gridDim.x) {
      uint32_t d = 0;
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const bool chunk_start = kt % kChunkSteps == 0;
        if (chunk_start) {
          const int cb = ch & 1;
          if (ch >= 2) mbar_wait(&tempty[cb], ((ch >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          d = tmem + (uint32_t)(cb * BN);
        }
        const int s = it % STAGES;
        mbar_wait(&conv[s], (it / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const float* st = stage0 + s * kStage;
          const float* ah = st;
          const float* al = st + kTile;
          const float* bh = st + 2 * kTile;
          const float* bl = st + 3 * kTile;
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint32_t acc0 = (!chunk_start || j > 0) ? 1u : 0u;
            mma_tf32(d, make_desc<A_MN>(ah, j), make_desc<B_MN>(bh, j), idesc, acc0);
            mma_tf32(d, make_desc<A_MN>(ah, j), make_desc<B_MN>(bl, j), idesc, 1u);
            mma_tf32(d, make_desc<A_MN>(al, j), make_desc<B_MN>(bh, j), idesc, 1u);
          }
          mma_commit(&empty[s]);                       // stage s is free once these complete
          if (kt % kChunkSteps == kChunkSteps - 1 || kt == KT - 1)
            mma_commit(&tfull[ch & 1]);                // this chunk's accumulator is complete
        }
        __syncwarp();
        if (kt % kChunkSteps == kChunkSteps - 1 || kt == KT - 1) ++ch;
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 12) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tmem));
  }
}

template <typename IDX, bool A_MN, bool B_MN>
static int launch_dir(const LaunchArgs& a, cudaStream_t s) {
  constexpr int smem = STAGES * kStage * (int)sizeof(float) + (3 * STAGES + 4) * 8 + 16;
  auto kern = tc_umma_f32_kernel<IDX, A_MN, B_MN>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return -1;
    attr = true;
  }
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int T = tiles_m * tiles_n;
  const int grid = T < a.num_sms ? T : a.num_sms;
  kern<<<grid, kThreads, smem, s>>>(
      static_cast<const float*>(a.A), static_cast<const float*>(a.B), static_cast<float*>(a.C),
      static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.M, a.N, a.K, tiles_m,
      tiles_n, a.alpha, a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace umma

// fp32 through the tensor cores (3xTF32). Applies to int32-offset fp32 contractions with
// K >= 1. Both operands are staged K-major: the MN-major (transposed) tf32 operand mode left
// the accumulator at zero on this part (tools/calib/umma_tf32_test.cu sweeps it), and the
// core-matrix lane mapping reads full 32-byte sectors from an M-contiguous operand anyway.
// 0 = not applicable, 1 = launched, -1 = CUDA error.
int launch_umma_f32(const LaunchArgs& a, cudaStream_t stream) {
  if (!a.f32 || a.idx64 || a.K < 1) return 0;
  return umma::launch_dir<int, false, false>(a, stream);
}

}  // namespace tcb
