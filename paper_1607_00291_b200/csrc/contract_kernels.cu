// sm_100a contraction kernel: block-scatter gather staging + FP64 tensor-core (DMMA) micro-kernel
// + scatter-aware alpha/beta epilogue. DESIGN.md §Kernels describes the design; the paper's
// counterparts are cited inline (PAPER.md = P:line).
//
// One CTA computes a kBM x kBN tile of the matricised C (a tile is a sub-range of the
// row and column scatter vectors, no data movement). The K loop is serial per tile.
// Per K step the CTA stages an A tile (kBM x kBK) and a B tile (kBK x kBN) from global memory
// into shared memory -- the GPU form of "packing" -- reading each element at
// base + rscat[i] + cscat[p] with cp.async. Where the block-scatter vector says two consecutive
// entries are consecutive addresses (block size 2) and the address is 16-byte
// aligned, one 16-byte cp.async moves both; otherwise two 8-byte gathers (the scatter path).
// Each operand is gathered along the bundle in which it has its unit stride (a_vec_m / b_vec_k),
// so warps read contiguous runs and the shared-memory layout follows that direction.
// The micro-kernel is mma.sync m16n8k4 f64 (SASS DMMA.8x8x4) over 64x32 warp tiles, and the
// epilogue writes alpha*acc + beta*C through rscat_C / cscat_C (beta == 0 never
// reads C).
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include "dev_common.cuh"
#include "kernels.hpp"

namespace tcb {
namespace {

constexpr int BM = kBM, BN = kBN, BK = kBK;
constexpr int NTHREADS = 256;             // 8 warps: 2 (M) x 4 (N), warp tile 64 x 32
constexpr int WM = 64, WN = 32;
constexpr int STAGES = 4;
constexpr int PAD = 4;                    // doubles; makes fragment loads bank-conflict free
constexpr int GROUP_M = 8;                // tile rasterisation: 8 M-tiles share B panels in L2

// shared-memory stage sizes (doubles) for each operand layout
constexpr int A_STAGE_VM = BK * (BM + PAD);   // As[k][m]   (gathered along M)
constexpr int A_STAGE_VK = BM * (BK + PAD);   // As[m][k]   (gathered along K)
constexpr int B_STAGE_VK = BN * (BK + PAD);   // Bs[n][k]
constexpr int B_STAGE_VN = BK * (BN + PAD);   // Bs[k][n]

template <bool A_VM> struct ALayout {
  static constexpr int STAGE = A_VM ? A_STAGE_VM : A_STAGE_VK;
  __device__ static __forceinline__ int at(int m, int k) {
    return A_VM ? k * (BM + PAD) + m : m * (BK + PAD) + k;
  }
};
template <bool B_VK> struct BLayout {
  static constexpr int STAGE = B_VK ? B_STAGE_VK : B_STAGE_VN;
  __device__ static __forceinline__ int at(int k, int n) {
    return B_VK ? n * (BK + PAD) + k : k * (BN + PAD) + n;
  }
};

using namespace dev;

// ------------------------------------------------------------------------------------------
// Operand loaders. A "pair" is two consecutive entries of the table the operand is gathered
// along; "rows" are entries of the other table. Each thread owns 4 pair slots per stage.
//
// Gather along the tile's fixed bundle (M for A, N for B): the pair is fixed for the whole
// K loop (offsets held in registers), the 4 rows are K entries that change every stage.
// Gather along K: the 4 rows are fixed (M or N entries), the pair is a K pair per stage.
// ------------------------------------------------------------------------------------------
template <typename IDX>
struct FixedPairLoader {   // pairs along the fixed (M/N) bundle, rows along K
  IDX o0, o1;              // fixed offsets of the pair
  bool vec, v0, v1;        // contiguous pair; entry validity
  IDX rowoff[4];           // prefetched K offsets for the next stage to issue
  int pcol;                // pair index 0..63 within the tile
  int rbase;               // first row (0..3)

  __device__ void init(const IDX* fixed_tab, const uint8_t* pairflag, int base, int extent,
                       int tid) {
    pcol = tid & 63;
    rbase = tid >> 6;
    int e = base + 2 * pcol;
    o0 = fixed_tab[e];
    o1 = fixed_tab[e + 1];
    v0 = e < extent;
    v1 = e + 1 < extent;
    vec = v1 && pairflag[e >> 1];
  }
  __device__ void prefetch(const IDX* ktab, int k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) rowoff[j] = __ldg(ktab + k0 + rbase + 4 * j);
  }
  // smem element index for (row r, pair col) in the [row][fixed] layout with row stride LD
  template <int LD>
  __device__ void issue(double* sm, const double* g, int k0, int K) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = rbase + 4 * j;
      bool kv = k0 + r < K;
      double* d = sm + r * LD + 2 * pcol;
      const double* p0 = g + (o0 + rowoff[j]);
      if (vec && kv && aligned16(p0)) {
        cp_async16(d, p0, true);
      } else {
        cp_async8(d, p0, kv && v0);
        cp_async8(d + 1, g + (o1 + rowoff[j]), kv && v1);
      }
    }
  }
};

template <typename IDX>
struct KPairLoader {       // pairs along K, rows along the fixed (M/N) bundle
  IDX rowoff[4];           // fixed offsets of the 4 rows
  unsigned rowvalid;       // bit j: row j in range
  IDX k0off, k1off;        // prefetched offsets of the K pair for the next stage
  bool kvec;
  int pk;                  // pair index 0..7
  int rbase;               // first row 0..31

  __device__ void init(const IDX* fixed_tab, int base, int extent, int tid) {
    pk = tid & 7;
    rbase = tid >> 3;
    rowvalid = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int e = base + rbase + 32 * j;
      rowoff[j] = fixed_tab[e];
      if (e < extent) rowvalid |= 1u << j;
    }
  }
  __device__ void prefetch(const IDX* ktab, const uint8_t* pairflag, int k0, int K) {
    int k = k0 + 2 * pk;
    k0off = __ldg(ktab + k);
    k1off = __ldg(ktab + k + 1);
    kvec = (k + 1 < K) && __ldg(pairflag + (k >> 1));
  }
  // [row][k] layout with row stride LD
  template <int LD>
  __device__ void issue(double* sm, const double* g, int k0, int K) {
    int k = k0 + 2 * pk;
    bool kv0 = k < K, kv1 = k + 1 < K;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int r = rbase + 32 * j;
      bool rv = (rowvalid >> j) & 1;
      double* d = sm + r * LD + 2 * pk;
      const double* p0 = g + (rowoff[j] + k0off);
      if (kvec && rv && aligned16(p0)) {
        cp_async16(d, p0, true);
      } else {
        cp_async8(d, p0, rv && kv0);
        cp_async8(d + 1, g + (rowoff[j] + k1off), rv && kv1);
      }
    }
  }
};

template <bool VEC_FIXED, typename IDX> struct LoaderSel;
template <typename IDX> struct LoaderSel<true, IDX> { using type = FixedPairLoader<IDX>; };
template <typename IDX> struct LoaderSel<false, IDX> { using type = KPairLoader<IDX>; };

// ------------------------------------------------------------------------------------------
// The kernel. A_VM: A gathered along M (else along K). B_VK: B gathered along K (else N).
// ------------------------------------------------------------------------------------------
template <typename IDX, bool A_VM, bool B_VK>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_dmma_f64_kernel(const double* __restrict__ A, const double* __restrict__ B,
                   double* __restrict__ C,
                   const IDX* __restrict__ rA, const IDX* __restrict__ cA,
                   const IDX* __restrict__ rB, const IDX* __restrict__ cB,
                   const IDX* __restrict__ rC, const IDX* __restrict__ cC,
                   const uint8_t* __restrict__ vA, const uint8_t* __restrict__ vB,
                   int M, int N, int K, int tiles_m, int tiles_n, double alpha, double beta) {
  extern __shared__ __align__(128) double smem[];
  using AL = ALayout<A_VM>;
  using BL = BLayout<B_VK>;
  double* As = smem;
  double* Bs = smem + STAGES * AL::STAGE;

  // grouped rasterisation of the tile grid (L2 reuse of A and B panels)
  const int pid = blockIdx.x;
  const int group_size = GROUP_M * tiles_n;
  const int first_m = (pid / group_size) * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int tm = first_m + (pid % group_size) % gm;
  const int tn = (pid % group_size) / gm;
  const int m0 = tm * BM, n0 = tn * BN;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * WM, wn = (warp >> 1) * WN;

  typename LoaderSel<A_VM, IDX>::type la;
  typename LoaderSel<B_VK == false, IDX>::type lb;
  if constexpr (A_VM) la.init(rA, vA, m0, M, tid); else la.init(rA, m0, M, tid);
  if constexpr (!B_VK) lb.init(cB, vB, n0, N, tid); else lb.init(cB, n0, N, tid);

  auto prefetch = [&](int kt) {
    int k0 = kt * BK;
    if constexpr (A_VM) la.prefetch(cA, k0); else la.prefetch(cA, vA, k0, K);
    if constexpr (!B_VK) lb.prefetch(rB, k0); else lb.prefetch(rB, vB, k0, K);
  };
  auto issue = [&](int kt) {
    int k0 = kt * BK;
    double* as = As + (kt % STAGES) * AL::STAGE;
    double* bs = Bs + (kt % STAGES) * BL::STAGE;
    if constexpr (A_VM) la.template issue<BM + PAD>(as, A, k0, K);
    else la.template issue<BK + PAD>(as, A, k0, K);
    if constexpr (!B_VK) lb.template issue<BN + PAD>(bs, B, k0, K);
    else lb.template issue<BK + PAD>(bs, B, k0, K);
  };

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) { prefetch(s); issue(s); }
    cp_async_commit();
  }
  if (STAGES - 1 < KT) prefetch(STAGES - 1);

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) {
        issue(nk);
        if (nk + 1 < KT) prefetch(nk + 1);
      }
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * AL::STAGE;
    const double* bs = Bs + (kt % STAGES) * BL::STAGE;
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
  }
  cp_async_wait<0>();

  // epilogue: C[rC[m] + cC[n]] = alpha*acc + beta*C  (beta == 0: C not read)
  IDX rc[8], cc[8];
  int mm[8], nn[8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int m = m0 + wm + 16 * i + g + 8 * h;
      mm[2 * i + h] = m;
      rc[2 * i + h] = rC[m];
    }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      int n = n0 + wn + 8 * j + 2 * t + e;
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
          double* p = C + (rc[2 * i + h] + cc[2 * j + e]);
          double v = alpha * acc[i][j][2 * h + e];
          if (beta != 0.0) v = fma(beta, *p, v);
          *p = v;
        }
    }
}

template <typename IDX, bool A_VM, bool B_VK>
int launch_f64(const LaunchArgs& a, cudaStream_t stream) {
  constexpr int smem =
      STAGES * (ALayout<A_VM>::STAGE + BLayout<B_VK>::STAGE) * (int)sizeof(double);
  auto kern = tc_dmma_f64_kernel<IDX, A_VM, B_VK>;
  static std::atomic<int> attr[kMaxDevices];
  if (!ensure_dyn_smem(kern, smem, attr)) return -1;
  int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n);
  kern<<<grid, NTHREADS, smem, stream>>>(
      static_cast<const double*>(a.A), static_cast<const double*>(a.B),
      static_cast<double*>(a.C), static_cast<const IDX*>(a.rA), static_cast<const IDX*>(a.cA),
      static_cast<const IDX*>(a.rB), static_cast<const IDX*>(a.cB),
      static_cast<const IDX*>(a.rC), static_cast<const IDX*>(a.cC), a.vA, a.vB, a.M, a.N, a.K,
      tiles_m, tiles_n, a.alpha, a.beta);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <typename IDX>
int dispatch_dir(const LaunchArgs& a, cudaStream_t s) {
  if (a.a_vec_m) return a.b_vec_k ? launch_f64<IDX, true, true>(a, s) : launch_f64<IDX, true, false>(a, s);
  return a.b_vec_k ? launch_f64<IDX, false, true>(a, s) : launch_f64<IDX, false, false>(a, s);
}

}  // namespace

// ws_<type>_a<mode>.cu: one translation unit per (element type, A gather mode)
int launch_ws_f64_a0(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f64_a1(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f64_a2(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f64_idx64(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_ffma_a0(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_ffma_a1(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_ffma_a2(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_ffma_idx64(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_ffma_a3(const LaunchArgs& a, cudaStream_t stream);
int launch_ws_f32_dmma(const LaunchArgs& a, cudaStream_t stream);   // ws_f32_dmma.cu

// Gather mode per operand: vectors when the plan proved every vector contiguous and aligned,
// else the coalesced element gather or the per-vector check, as the plan prefers.
static int launch_ws(const LaunchArgs& args, cudaStream_t stream) {
  LaunchArgs a = args;
  a.a_mode = a.a_vec_all ? 0 : (a.a_elem ? 2 : 1);
  a.b_mode = a.b_vec_all ? 0 : (a.b_elem ? 2 : 1);
  if (a.f32 && a.f32_dmma) return launch_ws_f32_dmma(a, stream);
  if (a.idx64) return a.f32 ? launch_ws_f32_ffma_idx64(a, stream) : launch_ws_f64_idx64(a, stream);
  if (a.f32) {
    // A and B both K-contiguous: transpose A into [k][m] while gathering (TC_FFMA_AT=0: off)
    if (!a.a_vec_m && a.b_vec_k && a.f32_a_transpose) return launch_ws_f32_ffma_a3(a, stream);
    switch (a.a_mode) {
      case 0: return launch_ws_f32_ffma_a0(a, stream);
      case 1: return launch_ws_f32_ffma_a1(a, stream);
      default: return launch_ws_f32_ffma_a2(a, stream);
    }
  }
  switch (a.a_mode) {
    case 0: return launch_ws_f64_a0(a, stream);
    case 1: return launch_ws_f64_a1(a, stream);
    default: return launch_ws_f64_a2(a, stream);
  }
}

// Kernel selection: the warp-specialised kernel (contract_ws.cu, fp64 and fp32) is the default;
// TC_KERNEL=simple selects the first (non-specialised, fp64-only) kernel for ablation.
// TC_KERNEL=ws_nosk keeps the persistent kernel but turns off its stream-K tail.
static int kernel_choice() {
  static int choice = [] {
    const char* e = getenv("TC_KERNEL");
    if (e && !strcmp(e, "simple")) return 1;
    if (e && !strcmp(e, "ws_nosk")) return 2;
    return 0;
  }();
  return choice;
}

// The skinny-contraction kernel (skinny.cu) runs for every skinny shape (measured against the
// tensor-core tile on the f2 strings, profiles/r01/suite_f2_skinny_ab.txt); TC_SKINNY=0 turns
// it off. Read on every call, so tests can switch it.
static int skinny_mode() {
  const char* e = getenv("TC_SKINNY");
  if (e && !strcmp(e, "0")) return 0;
  return 2;
}

// TC_RANKK=0 sends K <= 16 contractions with large free extents to the tile kernels instead
// of the rank-k kernel (rankk.cu). Read on every call (tests cover both paths).
static bool rankk_enabled() {
  const char* e = getenv("TC_RANKK");
  return !(e && !strcmp(e, "0"));
}

// TC_TINY=0 sends tiny contractions to the tensor-core kernel too (tests cover both paths).
static bool tiny_enabled() {
  const char* e = getenv("TC_TINY");
  return !(e && !strcmp(e, "0"));
}

// fp32 contractions run on the tcgen05 tensor cores as 3xTF32 (umma_f32.cu): 1.1-1.6x SGEMM on
// cfg4 against 0.7-0.95x for the FFMA2 kernel (profiles/r01/ab_f32_umma.txt). TC_F32_UMMA=0
// selects the FFMA2 kernel (contract_ws.cuh) instead. Read on every call (tests cover both).
static bool umma_f32_enabled() {
  const char* e = getenv("TC_F32_UMMA");
  return !(e && !strcmp(e, "0"));
}

int launch_contract(const LaunchArgs& args, cudaStream_t stream) {
  if (args.M <= 0 || args.N <= 0) return 0;
  const int choice = kernel_choice();
  if (choice == 0 && tiny_enabled()) {
    const int r = launch_tiny(args, stream);
    if (r != 0) return r;
  }
  if (choice == 0 && rankk_enabled()) {
    const int r = launch_rankk(args, stream);
    if (r != 0) return r;
  }
  if (choice == 0 && skinny_mode() != 0) {
    const int r = launch_skinny(args, stream, skinny_mode() == 2);
    if (r != 0) return r;
  }
  if (choice == 1 && !args.f32)
    return args.idx64 ? dispatch_dir<long long>(args, stream) : dispatch_dir<int>(args, stream);
  if (choice == 0 && args.f32 && umma_f32_enabled()) {
    // N = 256 form by default (TC_UMMA_FORM=128|256|pair forces a form): with the round-2
    // gather modes (one-line element gathers, pairs, B's N vectors through a [k][n] staging, A's
    // M vectors) it wins on every cfg4 case and on the GEMM-layout sweep (4096^3 141 -> 156
    // TF/s; profiles/r02/ab_umma_forms2.txt, ab_umma_am.txt)
    const char* fe = getenv("TC_UMMA_FORM");
    const bool n256 = fe ? !strcmp(fe, "256") : true;
    const bool pair = fe && !strcmp(fe, "pair");
    const int r = pair   ? launch_umma_f32_pair(args, stream)
                  : n256 ? launch_umma_f32_n256(args, stream)
                         : launch_umma_f32(args, stream);
    if (r != 0) return r;
  }
  LaunchArgs a = args;
  a.stream_k = args.stream_k && choice != 2;
  return launch_ws(a, stream);
}

}  // namespace tcb
