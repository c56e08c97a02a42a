// Persistent tile schedule shared by the tensor-core kernels (contract_ws.cuh, umma_f32.cu):
// data-parallel whole tiles plus a stream-K tail fixed up in place through per-tile flags.
#pragma once

#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

namespace tcb {
namespace sched {

// ------------------------------------------------------------------------------------------
// Persistent schedule: data-parallel full waves + a stream-K tail.
// Tiles [0, D) are whole tiles, dealt round-robin (CTA w takes w, w+P, ...), so CTAs running at
// the same time work on consecutive tiles (L2 reuse through the grouped rasterisation). The
// last S = T - D tiles are split by K iterations evenly over P_sk CTAs (stream-K), which removes
// the wave-quantisation loss of the final partial wave. Each CTA walks its stream-K range in
// REVERSE tile order, so the k-first piece of every split tile is computed at the start of the
// tail and its k-last piece at the end: the first piece writes alpha*acc + beta*C, later pieces
// add alpha*acc in a fixed order behind a per-tile flag. No partial-sum workspace, deterministic
// results, and a piece only waits on lower-ranked CTAs' first work items (no deadlock).
// ------------------------------------------------------------------------------------------
// Stream-K tail tiles that can carry work weights. Sched is a by-value kernel parameter: with 32
// (a 33-int prefix-sum array) the bench workload ran 0.7% slower than with 16 or fewer, though
// it never uses the weights (cfg5 2422 vs 2404-2405 ms, same box; profiles/r02/ab_sched_param.txt)
#ifndef TC_SK_MAXW
#define TC_SK_MAXW 16   // measurement override
#endif
constexpr int kMaxWeighted = TC_SK_MAXW;

struct Sched {
  int T, D, P, KT;          // tiles, data-parallel tiles, CTAs in the DP phase, K iterations
  int P_sk;                 // CTAs in the stream-K tail (0: no tail)
  long long I;              // stream-K iterations = (T - D) * KT
  // wave alignment of the data-parallel phase: before its j-th whole tile (j >= 1) a CTA's
  // producers wait (bounded) until the wave counter reaches wave_base + j * P, i.e. every CTA
  // has issued its loads of wave j - 1, so the CTAs of a wave walk K together and share the A
  // and B panels in L2 instead of drifting apart over hundreds of waves
  unsigned wave_base;
  int wave_sync;
  // stream-K flags carry this launch's epoch in their upper 24 bits (epoch << 8) and a piece
  // count in the low 8 bits: a value left behind by any earlier launch on the stream, finished
  // or aborted, never matches, so no per-launch reset is needed and none can be missed
  unsigned epoch;
  // Work-weighted stream-K (weighted != 0; the DMMA kernel on ragged few-tile shapes): tail tile
  // t costs w_t per K iteration (edge tiles skip empty MMAs and run faster), cum[t] = sum of
  // w_t' for t' < t. CTA w takes the K iterations whose work lies in [w W / P_sk,
  // (w + 1) W / P_sk), W = KT cum[T - D], instead of an equal number of iterations.
  int weighted;
  int cum[kMaxWeighted + 1];
  // Cluster split-K (csplit = S > 0; the DMMA kernel on few-tile problems): the grid is T x S
  // CTAs in clusters of S, cluster t computes tile t, its CTA of rank r the K iterations
  // [r KT / S, (r + 1) KT / S); the S partial tiles are summed through distributed shared
  // memory in rank order (no flags, no fix-up chain).
  int csplit;
};

// First stream-K iteration of CTA w (w = P_sk: the end).
__host__ __device__ inline long long sk_bound(const Sched& s, int w) {
  if (!s.weighted) return (long long)w * s.I / s.P_sk;
  const int n = s.T - s.D;
  const long long W = (long long)w * ((long long)s.KT * s.cum[n]) / s.P_sk;
  int t = 0;
  while (t + 1 < n && (long long)s.KT * s.cum[t + 1] <= W) ++t;
  const long long wt = s.cum[t + 1] - s.cum[t], off = W - (long long)s.KT * s.cum[t];
  return (long long)t * s.KT + (off + wt - 1) / wt;
}
// The CTA whose stream-K range holds iteration g.
__host__ __device__ inline int sk_owner(const Sched& s, long long g) {
  if (!s.weighted) return (int)(((g + 1) * s.P_sk + s.I - 1) / s.I) - 1;
  int lo = 0, hi = s.P_sk;   // the largest w with sk_bound(w) <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sk_bound(s, mid) <= g) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct WorkIter {
  int dp_t, D, P, KT;
  int sk_t, sk_lo;          // current / lowest stream-K tile (relative to D), descending
  int cs_kb, cs_ke;         // K range of a data-parallel item (cluster split-K: a share)
  long long g0, g1;         // this CTA's stream-K iteration range

  __device__ __forceinline__ void init(const Sched& s, int w) {
    D = s.D; P = s.P; KT = s.KT;
    if (s.csplit) {   // one item: tile w / S, the rank's share of K (as a data-parallel item)
      const int r = w % s.csplit;
      dp_t = w / s.csplit; D = dp_t + 1; P = 1;
      cs_kb = (int)((long long)r * KT / s.csplit);
      cs_ke = (int)((long long)(r + 1) * KT / s.csplit);
      sk_t = -1; sk_lo = 0; g0 = g1 = 0;
      return;
    }
    cs_kb = 0; cs_ke = KT;
    dp_t = w < s.P ? w : s.D;
    sk_t = -1; sk_lo = 0; g0 = g1 = 0;
    if (w < s.P_sk) {
      g0 = sk_bound(s, w);
      g1 = sk_bound(s, w + 1);
      if (g1 > g0) { sk_t = (int)((g1 - 1) / KT); sk_lo = (int)(g0 / KT); }
    }
  }
  // next work item: tile index, K-iteration range [kb, ke), stream-K piece flag
  __device__ __forceinline__ bool next(int& tile, int& kb, int& ke, bool& sk) {
    if (dp_t < D) { tile = dp_t; dp_t += P; kb = cs_kb; ke = cs_ke; sk = false; return true; }
    if (sk_t >= sk_lo) {
      const long long base = (long long)sk_t * KT;
      kb = (int)(g0 > base ? g0 - base : 0);
      ke = (int)(g1 - base < KT ? g1 - base : KT);
      tile = D + sk_t;
      --sk_t;
      sk = true;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Wait until a stream-K flag holds `target` (epoch | piece). A piece only waits for lower-ranked
// CTAs' first work items, so the wait is bounded by one piece's run time; past kFlagTimeoutNs
// something is broken (a CTA that never ran, corrupted flags) and the kernel traps instead of
// spinning forever: the launch fails with cudaErrorLaunchFailure / an illegal-instruction error.
constexpr unsigned long long kFlagTimeoutNs = 30ull * 1000000000ull;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static __device__ __noinline__ void flag_timeout(const int* flag, int target) {
  printf("tc_b200: stream-K fix-up flag timeout (block %d, flag %d, want %d)\n",
         (int)blockIdx.x, ld_acquire(flag), target);
  __trap();
}
__device__ __forceinline__ void wait_flag(const int* flag, int target) {
  if (ld_acquire(flag) == target) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire(flag) != target) {
    __nanosleep(64);
    if (global_ns() - t0 > kFlagTimeoutNs) flag_timeout(flag, target);
  }
}
// Pair form (two arrivals per piece, count_flag): wait until this launch's count reaches
// `target`. The two CTAs of a pair wait for the same count, and the first one through may add
// its own arrival before the other has looked, so the wait is for `>=`, not `==`.
__device__ __forceinline__ void wait_flag_ge(const int* flag, unsigned epoch, int target) {
  auto done = [&](unsigned v) { return (v & ~0xffu) == epoch && (int)(v & 0xffu) >= target; };
  if (done((unsigned)ld_acquire(flag))) return;
  const unsigned long long t0 = global_ns();
  while (!done((unsigned)ld_acquire(flag))) {
    __nanosleep(64);
    if (global_ns() - t0 > kFlagTimeoutNs) flag_timeout(flag, (int)(epoch | (unsigned)target));
  }
}
// Count one arrival on a flag of this launch's epoch: a value from another epoch counts as 0.
__device__ __forceinline__ void count_flag(int* flag, unsigned epoch) {
  int old = ld_acquire(flag);
  while (true) {
    const int nw = ((unsigned)old & ~0xffu) == epoch ? old + 1 : (int)(epoch | 1u);
    const int prev = atomicCAS(flag, old, nw);
    if (prev == old) break;
    old = prev;
  }
}

// Host side of the schedule: D whole tiles round-robin over P = #SMs CTAs, the rest split by
// K iterations over P_sk CTAs (each gets >= kMinSkIters iterations). TC_KERNEL=ws_nosk turns
// the tail off (all tiles data-parallel) for ablation.
constexpr int kMinSkIters = 8;
constexpr int kMaxPieces = 16;   // at most this many stream-K pieces per tile (fix-up chain)

inline Sched make_sched(int T, int KT, int nsm, bool allow_sk, int dp_pct = 88,
                        int min_sk_iters = kMinSkIters, int max_pieces = kMaxPieces) {
  Sched s{};
  s.T = T; s.KT = KT; s.P = nsm;
  // Which tiles are split: the last full wave and the partial wave (stream-K over 1-2 waves,
  // enough iterations per CTA for a short tail), unless the partial wave is >= 88% full, which
  // then runs data-parallel (its idle share is smaller than the cost of the split pieces'
  // extra epilogues). Measured on cfg4 (profiles/r01/ab_sk_policy.txt); the fp32 tcgen05
  // kernel passes dp_pct = 70 (profiles/r01/ab_umma_sk.txt), the DMMA kernel 101 since its
  // fix-ups add at L2 (profiles/r02/ab_dppct.txt).
  int D;
  const int rem = T % nsm;
  if (!allow_sk || KT == 0 || rem == 0 || rem * 100 >= dp_pct * nsm) D = T;
  else if (T < nsm) D = 0;
  else D = (T / nsm - 1) * nsm;
  s.D = D;
  s.I = (long long)(T - D) * KT;
  long long psk = s.I / min_sk_iters;   // each stream-K CTA gets >= min_sk_iters iterations
  if (psk < 1) psk = 1;
  if (psk > nsm) psk = nsm;
  if (psk > (long long)(T - D) * max_pieces) psk = (long long)(T - D) * max_pieces;
  s.P_sk = D < T ? (int)psk : 0;
  return s;
}

}  // namespace sched
}  // namespace tcb
