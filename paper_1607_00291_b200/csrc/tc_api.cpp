// C ABI (include/tc.h): validation, plan cache, device tables, host (end-to-end) path.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "kernels.hpp"
#include "plan.hpp"
#include "tc.h"

namespace tcb {

// NVTX ranges around the entry points and the host path's stages (visible in nsys / ncu
// --nvtx; a push/pop costs nanoseconds when no tool is attached).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

static thread_local std::string g_detail;

static int fail(int code, const std::string& detail) {
  g_detail = detail;
  return code;
}
static int fail(const Status& s) { return fail(s.code, s.detail); }
static int cuda_fail(cudaError_t e, const char* what) {
  return fail(TC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device copies of a plan's tables on one device.
struct DeviceTables {
  int device = -1;
  int num_sms = 148;
  void* tab[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  uint8_t* vA = nullptr;
  uint8_t* vB = nullptr;
  uint8_t* vZ = nullptr;   // all-zero flags as long as vA and vB (TC_FORCE_PATH=scatter)
  int* bsh_p = nullptr;    // shifted N-vector tables of B (fp32 gather mode 12), or null
  int* bsh_c = nullptr;
  ~DeviceTables() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (device >= 0) cudaSetDevice(device);
    for (auto& p : tab) cudaFree(p);
    cudaFree(vA);
    cudaFree(vB);
    cudaFree(vZ);
    cudaFree(bsh_p);
    cudaFree(bsh_c);
    if (cur >= 0) cudaSetDevice(cur);
  }
};

// Stream-K fix-up flags, one buffer of 2 * #SMs ints per (device, stream). Every launch tags its
// flag values with a fresh epoch (sched.cuh), so a buffer is reused without a reset and a launch
// that was aborted half-way cannot poison later ones; launches on one stream are ordered,
// launches on different streams use different buffers.
struct FlagKey {
  int device;
  cudaStream_t stream;
  bool operator<(const FlagKey& o) const {
    return device != o.device ? device < o.device : stream < o.stream;
  }
};
// After the flags, one int is the wave counter of the data-parallel phase: it only grows (each
// whole tile adds 1) and the host keeps its expected value per stream (`wave_base`).
struct StreamFlags {
  int* flags = nullptr;
  std::atomic<unsigned> wave_base{0};
  std::atomic<unsigned> epoch{0};   // stream-K flag epochs handed out (sched.cuh)
};
static std::mutex g_flags_mu;
static std::map<FlagKey, StreamFlags> g_flags;

static StreamFlags* stream_flags(int device, cudaStream_t s, int cap) {
  std::lock_guard<std::mutex> lk(g_flags_mu);
  auto it = g_flags.find({device, s});
  if (it != g_flags.end()) return &it->second;
  int* f = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&f), sizeof(int) * (size_t)(cap + 1)) != cudaSuccess)
    return nullptr;
  // zeroed on the legacy stream, then waited for: the first launch may come on any stream,
  // including a non-blocking one that is not ordered after the legacy stream
  if (cudaMemset(f, 0, sizeof(int) * (size_t)(cap + 1)) != cudaSuccess ||
      cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess) {
    cudaFree(f);
    return nullptr;
  }
  StreamFlags& sf = g_flags[{device, s}];
  sf.flags = f;
  return &sf;
}

// TC_WAVE_SYNC=0 turns off the wave alignment of the data-parallel phase (ablation).
static bool wave_sync() {
  static const bool f = [] {
    const char* e = getenv("TC_WAVE_SYNC");
    return !(e && !strcmp(e, "0"));
  }();
  return f;
}

Plan::~Plan() {
  for (auto* d : dev) delete d;
}

static int64_t padded(int64_t n) { return ((n + kTablePad - 1) / kTablePad + 1) * kTablePad; }

// Vector flags = block-scatter vector with block size V = 16 / element size,
// reduced to "this block of V entries is V consecutive addresses" (a short tail block is 0).
static std::vector<uint8_t> vec_flags(const std::vector<int64_t>& scat, int64_t padlen,
                                      int64_t V) {
  std::vector<int64_t> bs = block_scatter(scat, V);
  std::vector<uint8_t> f((size_t)(padlen / V + 1), 0);
  for (size_t i = 0; i < bs.size(); ++i)
    f[i] = (bs[i] == 1 && (int64_t)(i + 1) * V <= (int64_t)scat.size()) ? 1 : 0;
  return f;
}

template <typename IDX>
static cudaError_t upload_table(const std::vector<int64_t>& v, void** out) {
  int64_t n = padded((int64_t)v.size());
  std::vector<IDX> h((size_t)n, 0);
  for (size_t i = 0; i < v.size(); ++i) h[i] = (IDX)v[i];
  cudaError_t e = cudaMalloc(out, sizeof(IDX) * (size_t)n);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*out, h.data(), sizeof(IDX) * (size_t)n, cudaMemcpyHostToDevice);
}

static cudaError_t upload_bytes(const std::vector<uint8_t>& v, uint8_t** out) {
  cudaError_t e = cudaMalloc((void**)out, v.size() + 16);
  if (e != cudaSuccess) return e;
  cudaMemset(*out, 0, v.size() + 16);
  return cudaMemcpy(*out, v.data(), v.size(), cudaMemcpyHostToDevice);
}

// Shifted N-vector tables of an N-contiguous fp32 B (umma_f32.cu gather mode 12; the
// block-scatter decision of P:644-683 taken per run instead of per aligned vector). Per tile
// block of 128 columns, cscat_B splits into runs of consecutive addresses. Run j (first column
// s, length L, offset b = cscat_B[s], c = b mod 4) owns ceil((L + 6) / 4) 16-byte slots of the
// [k][n] staging, filled for K index k with the aligned blocks starting at
// (b - c) + (rscat_B[k] - rscat_B[k] mod 4) + 4 i, so column n of k lands at staging word
// 4 * first slot + c + (n - s) + rscat_B[k] mod 4: a per-column base plus a per-k shift.
// prod[tn][slot] = (b - c + 4 i, L << 12 | (c - 4 i + 2048)) (block i of the run; unused slots
// (0, 1948): never copied); conv[tn][n] = 4 * first slot + c + (n - s). False when some tile
// block needs more than kShiftSlots slots (short runs: the element gathers are as good) or an
// offset does not fit the int32 tables.
static constexpr int kShiftSlots = 64;
static bool nshift_tables(const std::vector<int64_t>& cB, std::vector<int>& prod,
                          std::vector<int>& conv) {
  const int64_t N = (int64_t)cB.size();
  const int64_t tiles = (N + 127) / 128;
  prod.assign((size_t)(tiles * kShiftSlots * 2), 0);
  conv.assign((size_t)(tiles * 128), 0);
  for (int64_t t = 0; t < tiles; ++t) {
    const int64_t n0 = t * 128, n1 = std::min(N, n0 + 128);
    int slot = 0;
    for (int64_t n = n0; n < n1;) {
      int64_t e = n + 1;
      while (e < n1 && cB[(size_t)e] == cB[(size_t)(e - 1)] + 1) ++e;
      const int64_t L = e - n, nb = (L + 9) / 4;
      if (slot + nb > kShiftSlots) return false;
      const int64_t b = cB[(size_t)n], c = b & 3;
      if (b < INT32_MIN / 2 || b > INT32_MAX / 2) return false;
      for (int64_t i = 0; i < nb; ++i) {
        prod[(size_t)((t * kShiftSlots + slot + i) * 2)] = (int)(b - c + 4 * i);
        prod[(size_t)((t * kShiftSlots + slot + i) * 2 + 1)] = (int)((L << 12) | (c - 4 * i + 2048));
      }
      for (int64_t j = 0; j < L; ++j) conv[(size_t)(n + j)] = (int)(4 * slot + c + j);
      slot += (int)nb;
      n = e;
    }
    for (int i = slot; i < kShiftSlots; ++i)
      prod[(size_t)((t * kShiftSlots + i) * 2 + 1)] = 2048 - 100;   // L = 0: never copied
  }
  return true;
}

// The switches below are read on every call (a getenv per call costs well under a microsecond),
// so tests and ablations can flip them within one process.
//
// TC_FORCE_PATH=scatter: ablation of the block-scatter fast paths (the paper's SMTC):
// every vector flag is 0 and no operand is treated as vectorisable, so every element is an
// individual gather through the scatter vectors. TC_FORCE_PATH=blockscatter: every operand that
// is not proven all-vector takes the per-vector block-scatter check (gather mode 1)
// instead of the plan's choice.
static int force_path() {
  const char* e = getenv("TC_FORCE_PATH");
  if (e && !strcmp(e, "scatter")) return 1;
  if (e && !strcmp(e, "blockscatter")) return 2;
  return 0;
}
static bool force_scatter() { return force_path() == 1; }

// TC_F32_MMA=dmma: fp32 contractions through the DMMA micro-kernel (fp64 accumulation, one
// rounding) instead of the default FFMA micro-kernel (fp32 accumulation).
static bool f32_dmma() {
  const char* e = getenv("TC_F32_MMA");
  return e && !strcmp(e, "dmma");
}

// TC_GATHER=mixed|elem forces the gather mode of operands that are not all-vector (ablation);
// by default the plan decides (Plan::a_elem / b_elem).
static int gather_override() {
  if (force_path() == 2) return 1;
  const char* e = getenv("TC_GATHER");
  if (e && !strcmp(e, "mixed")) return 1;
  if (e && !strcmp(e, "elem")) return 2;
  return 0;
}

// Size limits of the tiny-contraction kernel (log2 of C elements and of multiply-adds);
// TC_TINY_LIMITS="mn,mnk" overrides them (tuning experiments).
static void tiny_limits(int* mn, int* mnk) {
  static int lim[2] = {-1, -1};
  if (lim[0] < 0) {
    lim[0] = 18; lim[1] = 24;
    const char* e = getenv("TC_TINY_LIMITS");
    if (e) std::sscanf(e, "%d,%d", &lim[0], &lim[1]);
  }
  *mn = lim[0];
  *mnk = lim[1];
}

static bool f32_a_transpose() {
  const char* e = getenv("TC_FFMA_AT");
  return !(e && !strcmp(e, "0"));
}

// Shifted N vectors for B (gather mode 12): TC_UMMA_SHIFT=0 never, 2 wherever the tables exist
// (tests, measurement), default (1) where the kernel selects them (umma_f32.cu); read per call
static int b_shift_mode() {
  const char* e = getenv("TC_UMMA_SHIFT");
  return e ? atoi(e) : 1;
}

static int get_tables(const Plan& p, DeviceTables** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(p.mu);
  for (auto* d : p.dev)
    if (d->device == dev) { *out = d; return TC_OK; }
  auto* d = new DeviceTables();
  d->device = dev;
  cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, dev);
  for (int i = 0; i < 6; ++i) {
    e = p.idx64 ? upload_table<long long>(p.kscat[i], &d->tab[i])
                : upload_table<int>(p.kscat[i], &d->tab[i]);
    if (e != cudaSuccess) { delete d; return cuda_fail(e, "table upload"); }
  }
  // A is gathered along rscat_A (M) or cscat_A (K); B along rscat_B (K) or cscat_B (N).
  const std::vector<int64_t>& ta = p.a_vec_m ? p.kscat[0] : p.kscat[1];
  const std::vector<int64_t>& tb = p.b_vec_k ? p.kscat[2] : p.kscat[3];
  const int64_t V = p.dtype == TC_F64 ? 2 : 4;
  std::vector<uint8_t> fa = vec_flags(ta, padded((int64_t)ta.size()), V);
  std::vector<uint8_t> fb = vec_flags(tb, padded((int64_t)tb.size()), V);
  e = upload_bytes(fa, &d->vA);
  if (e == cudaSuccess) e = upload_bytes(fb, &d->vB);
  if (e == cudaSuccess)
    e = upload_bytes(std::vector<uint8_t>(std::max(fa.size(), fb.size()), 0), &d->vZ);
  if (e == cudaSuccess && p.dtype == TC_F32 && !p.idx64 && !p.b_vec_k) {
    std::vector<int> prod, conv;
    if (nshift_tables(p.kscat[3], prod, conv)) {
      e = cudaMalloc(reinterpret_cast<void**>(&d->bsh_p), sizeof(int) * prod.size());
      if (e == cudaSuccess)
        e = cudaMemcpy(d->bsh_p, prod.data(), sizeof(int) * prod.size(), cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = cudaMalloc(reinterpret_cast<void**>(&d->bsh_c), sizeof(int) * conv.size());
      if (e == cudaSuccess)
        e = cudaMemcpy(d->bsh_c, conv.data(), sizeof(int) * conv.size(), cudaMemcpyHostToDevice);
    }
  }
  // the uploads ran on the legacy stream (a pageable cudaMemcpy may return before its DMA has
  // landed, cudaMemset is asynchronous): wait for them before any stream may read the tables
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
  if (e != cudaSuccess) { delete d; return cuda_fail(e, "flag upload"); }
  p.dev.push_back(d);
  *out = d;
  return TC_OK;
}

static int execute(const Plan& p, double alpha, const void* A, const void* B, double beta,
                   void* C, cudaStream_t stream) {
  if (p.empty_out || p.m == 0 || p.n == 0) return TC_OK;
  if (!C) return fail(TC_ERR_ARG, "null C");
  bool skip_ab = (alpha == 0.0) || p.k == 0;
  if (!skip_ab && (!A || !B)) return fail(TC_ERR_ARG, "null A or B");
  size_t esz = p.dtype == TC_F64 ? 8 : 4;
  for (const void* q : {A, B, (const void*)C})
    if (q && (reinterpret_cast<uintptr_t>(q) % esz) != 0)
      return fail(TC_ERR_ARG, "data pointer not aligned to the element size");
  DeviceTables* d = nullptr;
  int rc = get_tables(p, &d);
  if (rc != TC_OK) return rc;
  LaunchArgs a{};
  a.A = p.b.swapped ? B : A;  // after heuristic step 4 the roles of A and B are exchanged
  a.B = p.b.swapped ? A : B;
  a.C = C;
  a.rA = d->tab[0]; a.cA = d->tab[1]; a.rB = d->tab[2];
  a.cB = d->tab[3]; a.rC = d->tab[4]; a.cC = d->tab[5];
  const bool scatter_only = force_scatter();
  a.vA = scatter_only ? d->vZ : d->vA;
  a.vB = scatter_only ? d->vZ : d->vB;
  a.M = (int)p.m; a.N = (int)p.n; a.K = skip_ab ? 0 : (int)p.k;
  a.alpha = alpha; a.beta = beta;
  a.a_vec_m = p.a_vec_m; a.b_vec_k = p.b_vec_k; a.idx64 = p.idx64; a.f32 = p.dtype == TC_F32;
  a.a_vec_all = p.a_pairs_all && (reinterpret_cast<uintptr_t>(a.A) % 16) == 0 && !scatter_only;
  a.b_vec_all = p.b_pairs_all && (reinterpret_cast<uintptr_t>(a.B) % 16) == 0 && !scatter_only;
  a.a_vec2_all = p.a_pairs2_all && (reinterpret_cast<uintptr_t>(a.A) % 8) == 0 && !scatter_only;
  a.b_vec2_all = p.b_pairs2_all && (reinterpret_cast<uintptr_t>(a.B) % 8) == 0 && !scatter_only;
  a.bsh_p = d->bsh_p;
  a.bsh_c = d->bsh_c;
  a.b_shift = d->bsh_p != nullptr && (reinterpret_cast<uintptr_t>(a.B) % 16) == 0 &&
              !scatter_only ? b_shift_mode() : 0;
  a.a_elem = gather_override() ? gather_override() == 2 : p.a_elem;
  a.b_elem = gather_override() ? gather_override() == 2 : p.b_elem;
  a.f32_a_transpose = f32_a_transpose() && !scatter_only;
  a.c_lanes_n = p.c_unit_n;
  a.skinny_bu = p.skinny_bu;
  tiny_limits(&a.tiny_mn_log2, &a.tiny_mnk_log2);
  a.skinny_bv = p.skinny_bv;
  a.num_sms = d->num_sms;
  a.flags_cap = 2 * d->num_sms;
  StreamFlags* sf = stream_flags(d->device, stream, a.flags_cap);
  a.flags = sf ? sf->flags : nullptr;
  a.wave_base = sf ? &sf->wave_base : nullptr;
  if (sf) {
    // epochs 1 .. 2^24 - 1 (sched.cuh); when they wrap, the flags are zeroed on the stream
    // first, so a value from 2^24 launches ago cannot match
    const unsigned n = sf->epoch.fetch_add(1, std::memory_order_relaxed);
    const unsigned ep = n % 0xFFFFFFu + 1u;
    if (ep == 1u && n != 0u) {
      cudaError_t e = cudaMemsetAsync(sf->flags, 0, sizeof(int) * (size_t)a.flags_cap, stream);
      if (e != cudaSuccess) return cuda_fail(e, "flag reset");
    }
    a.flag_epoch = ep << 8;
  }
  a.wave_sync = sf != nullptr && wave_sync();
  a.stream_k = a.flags != nullptr;
  a.f32_dmma = f32_dmma();
  if (a.K == 0) { a.A = a.C; a.B = a.C; }  // never dereferenced
  int n = launch_contract(a, stream);
  if (n < 0) return cuda_fail(cudaGetLastError(), "kernel launch");
  return TC_OK;
}

// ---- plan cache --------------------------------------------------------------------------

static std::mutex g_cache_mu;
static std::map<std::string, std::shared_ptr<Plan>> g_cache;

static void key_tensor(std::string& k, const tc_tensor& t) {
  k.append(reinterpret_cast<const char*>(&t.rank), sizeof(t.rank));
  if (t.rank > 0) {
    k.append(reinterpret_cast<const char*>(t.lens), sizeof(int64_t) * (size_t)t.rank);
    k.append(reinterpret_cast<const char*>(t.strides), sizeof(int64_t) * (size_t)t.rank);
    k.append(t.labels, (size_t)t.rank);
  }
  k.push_back('|');
}

static int check_tensor(const tc_tensor* t, const char* name) {
  if (!t) return fail(TC_ERR_ARG, std::string("null tensor ") + name);
  if (t->rank < 0) return fail(TC_ERR_ARG, std::string("negative rank in ") + name);
  if (t->rank > TC_MAX_RANK) return fail(TC_ERR_UNSUPPORTED, std::string("rank > TC_MAX_RANK in ") + name);
  if (t->rank > 0 && (!t->lens || !t->strides || !t->labels))
    return fail(TC_ERR_ARG, std::string("null lens/strides/labels in ") + name);
  return TC_OK;
}

static int get_plan(tc_dtype dtype, const tc_tensor* A, const tc_tensor* B, const tc_tensor* C,
                    std::shared_ptr<Plan>* out) {
  Nvtx range("tc_plan_lookup");
  int rc;
  if ((rc = check_tensor(A, "A")) || (rc = check_tensor(B, "B")) || (rc = check_tensor(C, "C")))
    return rc;
  std::string key(1, (char)dtype);
  key_tensor(key, *A); key_tensor(key, *B); key_tensor(key, *C);
  for (const char* ov : {"TC_SKINNY_BV", "TC_SKINNY_BU"})   // planner overrides (plan.cpp)
    if (const char* e = getenv(ov)) { key.append(ov); key.append(e); }
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) { *out = it->second; return TC_OK; }
  }
  auto p = std::make_shared<Plan>();
  Status st = build_plan(dtype, *A, *B, *C, p.get());
  if (!st) return fail(st);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cache.size() > 4096) g_cache.clear();
  g_cache.emplace(key, p);
  *out = p;
  return TC_OK;
}

// C must not overlap A or B (reading R7): conservative byte-interval test.
static bool overlaps(const tc_tensor* X, const tc_tensor* C, size_t esz) {
  int64_t xl, xh, cl, ch;
  span(X->rank, X->lens, X->strides, &xl, &xh);
  span(C->rank, C->lens, C->strides, &cl, &ch);
  if (xl > xh || cl > ch || !X->data || !C->data) return false;
  const char* x0 = static_cast<const char*>(X->data) + xl * (int64_t)esz;
  const char* x1 = static_cast<const char*>(X->data) + (xh + 1) * (int64_t)esz;
  const char* c0 = static_cast<const char*>(C->data) + cl * (int64_t)esz;
  const char* c1 = static_cast<const char*>(C->data) + (ch + 1) * (int64_t)esz;
  return x0 < c1 && c0 < x1;
}

// ---- end-to-end path on host buffers (tc_contract_host) ------------------------------------
// The work is cut into chunks along one free label x of C (a contiguous range of x per chunk,
// a free sub-block of C is an independent contraction whose operands are strided
// sub-views). Host->device copies of chunk i+1, the contraction of chunk i and the
// device->host copy of chunk i-1 run on three streams at once, so the PCIe transfers hide
// behind the kernel. x is chosen so that C's chunks are disjoint address intervals (x has the
// largest stride of C) and the bytes copied are minimal; when no label qualifies, one chunk.
// Device staging buffers are kept per device between calls (tc_release_staging frees them).
struct Staging {
  void* buf[3] = {nullptr, nullptr, nullptr};
  size_t cap[3] = {0, 0, 0};
  cudaStream_t h2d = nullptr, d2h = nullptr;
};
static std::mutex g_stage_mu;
static std::map<int, Staging> g_stage;

static cudaError_t stage_reserve(Staging& st, int t, size_t bytes) {
  if (st.cap[t] >= bytes) return cudaSuccess;
  if (st.buf[t]) { cudaFree(st.buf[t]); st.buf[t] = nullptr; st.cap[t] = 0; }
  cudaError_t e = cudaMalloc(&st.buf[t], bytes);
  if (e == cudaSuccess) st.cap[t] = bytes;
  return e;
}

static int label_pos(const tc_tensor* T, char x) {
  for (int d = 0; d < T->rank; ++d)
    if (T->labels[d] == x) return d;
  return -1;
}

// Chunks along dimension `pos` are disjoint address intervals: a positive stride larger than
// the span of all other dimensions.
static bool outer_dim(const tc_tensor* T, int pos) {
  const int64_t s = T->strides[pos];
  if (s <= 0) return false;
  int64_t ext = 0;
  for (int d = 0; d < T->rank; ++d)
    if (d != pos) ext += (T->strides[d] < 0 ? -T->strides[d] : T->strides[d]) * (T->lens[d] - 1);
  return s > ext;
}

struct Piece {           // the address span [lo, hi] (elements, relative to data) of a sub-view
  int64_t lo = 1, hi = 0;
  int64_t bytes(size_t esz) const { return lo <= hi ? (hi - lo + 1) * (int64_t)esz : 0; }
};

// Span of T restricted to x in [x0, x0 + len) along dimension pos (pos < 0: whole tensor).
static Piece piece_of(const tc_tensor* T, int pos, int64_t x0, int64_t len) {
  Piece p;
  int64_t lens[TC_MAX_RANK];
  for (int d = 0; d < T->rank; ++d) lens[d] = T->lens[d];
  int64_t off = 0;
  if (pos >= 0) { lens[pos] = len; off = x0 * T->strides[pos]; }
  span(T->rank, lens, T->strides, &p.lo, &p.hi);
  if (p.lo <= p.hi) { p.lo += off; p.hi += off; }
  return p;
}

// chunks of the host path: 8 (TC_HOST_CHUNKS overrides, measurement)
static int host_chunks() {
  const char* e = getenv("TC_HOST_CHUNKS");
  const int n = e ? atoi(e) : 8;
  return n < 1 ? 1 : (n > 64 ? 64 : n);
}
constexpr int64_t kHostChunkMinBytes = 64ll << 20;

static int contract_host(tc_dtype dtype, double alpha, const tc_tensor* A, const tc_tensor* B,
                         double beta, const tc_tensor* C, cudaStream_t s) {
  Nvtx range("tc_contract_host");
  const int kHostChunks = host_chunks();
  std::shared_ptr<Plan> full;
  int rc = get_plan(dtype, A, B, C, &full);
  if (rc != TC_OK) return rc;
  const size_t esz = dtype == TC_F64 ? 8 : 4;
  if (overlaps(A, C, esz) || overlaps(B, C, esz)) return fail(TC_ERR_ALIAS, "C overlaps A or B");
  if (full->empty_out) return TC_OK;
  const bool need_ab = alpha != 0.0 && full->k > 0;
  const tc_tensor* T[3] = {A, B, C};
  for (int t = 0; t < 3; ++t)
    if ((t == 2 || need_ab) && !T[t]->data) return fail(TC_ERR_ARG, "null host data pointer");
  int64_t nC = 1;
  for (int d = 0; d < C->rank; ++d) nC *= C->lens[d];
  Piece whole[3];
  for (int t = 0; t < 3; ++t) whole[t] = piece_of(T[t], -1, 0, 0);
  // C is uploaded when it is read (beta != 0) or when its span has holes that must survive
  auto c_upload = [&](const Piece& pc, int64_t elems) {
    return beta != 0.0 || (pc.lo <= pc.hi && pc.hi - pc.lo + 1 != elems);
  };
  const int64_t unsplit = (need_ab ? whole[0].bytes(esz) + whole[1].bytes(esz) : 0) +
                          whole[2].bytes(esz) * (c_upload(whole[2], nC) ? 2 : 1);

  // -- choose the chunk label x (in C and in exactly one operand X; Y is the other operand)
  int best_c = -1, best_x = -1, best_t = -1;
  int64_t best_q = 0, best_cost = 0, best_len = 0;
  if (need_ab && unsplit >= kHostChunkMinBytes) {
    for (int pc = 0; pc < C->rank; ++pc) {
      const int64_t len = C->lens[pc];
      if (len < 2 || !outer_dim(C, pc)) continue;
      const int xt = label_pos(A, C->labels[pc]) >= 0 ? 0 : 1;
      const int px = label_pos(T[xt], C->labels[pc]);
      if (px < 0) continue;
      const int64_t q = (len + kHostChunks - 1) / kHostChunks;
      int64_t cost = whole[1 - xt].bytes(esz);
      for (int64_t x0 = 0; x0 < len; x0 += q) {
        const int64_t l = std::min(q, len - x0);
        const Piece pcx = piece_of(C, pc, x0, l);
        cost += piece_of(T[xt], px, x0, l).bytes(esz) +
                pcx.bytes(esz) * (c_upload(pcx, nC / len * l) ? 2 : 1);
      }
      if (cost * 20 > unsplit * 21) continue;  // more than 5% extra copy volume
      if (best_c < 0 || cost < best_cost || (cost == best_cost && len > best_len)) {
        best_c = pc; best_x = px; best_t = xt; best_q = q; best_cost = cost; best_len = len;
      }
    }
  }
  const int nch = best_c < 0 ? 1 : (int)((best_len + best_q - 1) / best_q);

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging& st = g_stage[dev];
  if (!st.h2d) {
    if ((e = cudaStreamCreateWithFlags(&st.h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&st.d2h, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream creation");
  }
  const char* dbase[3] = {nullptr, nullptr, nullptr};
  for (int t = 0; t < 3; ++t) {
    if ((t < 2 && !need_ab) || whole[t].lo > whole[t].hi) continue;
    if ((e = stage_reserve(st, t, (size_t)whole[t].bytes(esz))) != cudaSuccess)
      return cuda_fail(e, "staging allocation");
    dbase[t] = static_cast<const char*>(st.buf[t]) - whole[t].lo * (int64_t)esz;
  }
  auto h2d = [&](int t, const Piece& p) {
    if (p.lo > p.hi) return cudaSuccess;
    return cudaMemcpyAsync(const_cast<char*>(dbase[t]) + p.lo * (int64_t)esz,
                           static_cast<const char*>(T[t]->data) + p.lo * (int64_t)esz,
                           (size_t)p.bytes(esz), cudaMemcpyHostToDevice, st.h2d);
  };

  std::vector<cudaEvent_t> ev;
  auto event = [&](cudaEvent_t* out) {
    cudaError_t r = cudaEventCreateWithFlags(out, cudaEventDisableTiming);
    if (r == cudaSuccess) ev.push_back(*out);
    return r;
  };
  cudaEvent_t e_start = nullptr, e_y = nullptr, e_end = nullptr;
  std::vector<cudaEvent_t> e_in((size_t)nch, nullptr), e_out((size_t)nch, nullptr);
  if ((e = event(&e_start)) == cudaSuccess && (e = event(&e_y)) == cudaSuccess)
    e = event(&e_end);
  for (int i = 0; i < nch && e == cudaSuccess; ++i)
    if ((e = event(&e_in[(size_t)i])) == cudaSuccess) e = event(&e_out[(size_t)i]);
  // work already queued on `stream` (e.g. the producer of the host inputs) comes first
  if (e == cudaSuccess) e = cudaEventRecord(e_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st.h2d, e_start, 0);
  // Y (the operand without x) is needed by every chunk. When Y has a bound label y whose
  // chunks are contiguous (its outermost stride), the first chunk is itself computed as a sum
  // over up to 8 y-pieces (beta on the first piece, 1 after), so Y streams in behind that
  // chunk's kernels instead of being uploaded before the first one; otherwise Y goes up first.
  const int yt = best_c < 0 ? -1 : 1 - best_t;
  int py = -1, pxy = -1;
  int64_t ylen = 0, yq = 0;
  if (yt >= 0) {
    const tc_tensor* Y = T[yt];
    for (int d = 0; d < Y->rank && py < 0; ++d) {
      const int px = label_pos(T[best_t], Y->labels[d]);
      if (px >= 0 && Y->lens[d] >= 2 && outer_dim(Y, d)) { py = d; pxy = px; }
    }
    if (py >= 0) { ylen = Y->lens[py]; yq = (ylen + kHostChunks - 1) / kHostChunks; }
  }
  const int nyp = py < 0 ? 0 : (int)((ylen + yq - 1) / yq);
  std::vector<cudaEvent_t> e_ypc((size_t)nyp, nullptr);
  for (int j = 0; j < nyp && e == cudaSuccess; ++j) e = event(&e_ypc[(size_t)j]);
  if (e == cudaSuccess && yt >= 0 && py < 0) e = h2d(yt, whole[yt]);
  if (e == cudaSuccess) e = cudaEventRecord(e_y, st.h2d);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, e_y, 0);

  // the sub-contraction with x in [x0, x0 + l) and (ly > 0) y in [y0, y0 + ly)
  auto run = [&](int64_t x0, int64_t l, int64_t y0, int64_t ly, double beta_eff) {
    int64_t lens[3][TC_MAX_RANK];
    tc_tensor sub[3];
    int64_t off[3] = {0, 0, 0};
    for (int t = 0; t < 3; ++t) {
      sub[t] = *T[t];
      for (int d = 0; d < T[t]->rank; ++d) lens[t][d] = T[t]->lens[d];
      sub[t].lens = lens[t];
      const int pos = best_c < 0 ? -1 : (t == 2 ? best_c : (t == best_t ? best_x : -1));
      if (pos >= 0) { lens[t][pos] = l; off[t] += x0 * T[t]->strides[pos]; }
      const int ypos = ly <= 0 ? -1 : (t == yt ? py : (t == best_t ? pxy : -1));
      if (ypos >= 0) { lens[t][ypos] = ly; off[t] += y0 * T[t]->strides[ypos]; }
    }
    std::shared_ptr<Plan> p = full;
    if (best_c >= 0) {
      const int r = get_plan(dtype, &sub[0], &sub[1], &sub[2], &p);
      if (r != TC_OK) return r;
    }
    const char* dp[3];
    for (int t = 0; t < 3; ++t) dp[t] = dbase[t] ? dbase[t] + off[t] * (int64_t)esz : nullptr;
    return execute(*p, alpha, dp[0], dp[1], beta_eff, const_cast<char*>(dp[2]), s);
  };

  for (int i = 0; i < nch && e == cudaSuccess && rc == TC_OK; ++i) {
    Nvtx chunk_range("tc_contract_host chunk (H2D, kernels, D2H enqueue)");
    const int64_t x0 = i * best_q, l = best_c < 0 ? 0 : std::min(best_q, best_len - x0);
    // the chunk's address spans: x restricted to [x0, x0 + l)
    Piece pp[3];
    int64_t nCi = 1;
    for (int t = 0; t < 3; ++t) {
      const int pos = best_c < 0 ? -1 : (t == 2 ? best_c : (t == best_t ? best_x : -1));
      pp[t] = piece_of(T[t], pos, x0, l);
    }
    for (int d = 0; d < C->rank; ++d) nCi *= d == best_c ? l : C->lens[d];
    if (best_c < 0) {
      if (need_ab) {
        if ((e = h2d(0, pp[0])) != cudaSuccess || (e = h2d(1, pp[1])) != cudaSuccess) break;
      }
    } else if ((e = h2d(best_t, pp[best_t])) != cudaSuccess) {
      break;
    }
    if (c_upload(pp[2], nCi) && (e = h2d(2, pp[2])) != cudaSuccess) break;
    if ((e = cudaEventRecord(e_in[(size_t)i], st.h2d)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(s, e_in[(size_t)i], 0)) != cudaSuccess) break;
    if (i == 0 && nyp > 0) {
      for (int j = 0; j < nyp && e == cudaSuccess && rc == TC_OK; ++j) {
        const int64_t y0 = j * yq, ly = std::min(yq, ylen - y0);
        if ((e = h2d(yt, piece_of(T[yt], py, y0, ly))) != cudaSuccess) break;
        if ((e = cudaEventRecord(e_ypc[(size_t)j], st.h2d)) != cudaSuccess) break;
        if ((e = cudaStreamWaitEvent(s, e_ypc[(size_t)j], 0)) != cudaSuccess) break;
        rc = run(x0, l, y0, ly, j == 0 ? beta : 1.0);
      }
      if (e != cudaSuccess || rc != TC_OK) break;
    } else if ((rc = run(x0, l, 0, 0, beta)) != TC_OK) {
      break;
    }
    if ((e = cudaEventRecord(e_out[(size_t)i], s)) != cudaSuccess) break;
    if ((e = cudaStreamWaitEvent(st.d2h, e_out[(size_t)i], 0)) != cudaSuccess) break;
    if (pp[2].lo <= pp[2].hi)
      e = cudaMemcpyAsync(static_cast<char*>(C->data) + pp[2].lo * (int64_t)esz,
                          dbase[2] + pp[2].lo * (int64_t)esz, (size_t)pp[2].bytes(esz),
                          cudaMemcpyDeviceToHost, st.d2h);
  }
  // `stream` completes after the last copy back, whatever happened above
  cudaError_t e2 = cudaEventRecord(e_end, st.d2h);
  if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(s, e_end, 0);
  cudaError_t e3 = cudaStreamSynchronize(st.h2d);
  cudaError_t e4 = cudaStreamSynchronize(st.d2h);
  cudaError_t e5 = cudaStreamSynchronize(s);
  for (auto x : ev) cudaEventDestroy(x);
  if (e != cudaSuccess) return cuda_fail(e, "host path copy");
  if (rc != TC_OK) return rc;
  for (cudaError_t x : {e2, e3, e4, e5})
    if (x != cudaSuccess) return cuda_fail(x, "host path synchronize");
  return TC_OK;
}

}  // namespace tcb

using namespace tcb;

extern "C" {

// Restrict the bound label `lbl` of an operand to [lo, lo + len): same strides, shorter length,
// data pointer moved to element lo along it (a zero-copy sub-view).
static tc_tensor restrict_label(const tc_tensor* T, char lbl, int64_t lo, int64_t len, size_t esz,
                                std::vector<int64_t>& lens) {
  tc_tensor out = *T;
  lens.assign(T->lens, T->lens + T->rank);
  char* base = static_cast<char*>(T->data);
  for (int d = 0; d < T->rank; ++d)
    if (T->labels[d] == lbl) {
      lens[(size_t)d] = len;
      if (base) base += lo * T->strides[d] * (int64_t)esz;
    }
  out.lens = lens.data();
  out.data = base;
  return out;
}

int tc_contract(tc_dtype dtype, double alpha, const tc_tensor* A, const tc_tensor* B,
                double beta, const tc_tensor* C, void* stream) {
  Nvtx range("tc_contract");
  std::shared_ptr<Plan> p;
  int rc = get_plan(dtype, A, B, C, &p);
  if (rc != TC_OK) return rc;
  size_t esz = dtype == TC_F64 ? 8 : 4;
  if (overlaps(A, C, esz) || overlaps(B, C, esz))
    return fail(TC_ERR_ALIAS, "C overlaps A or B");
  if (p->split_label && alpha != 0.0 && !p->empty_out && p->k > 0 && !force_scatter()) {
    // sub-division blocked by a length with no small power-of-two divisor (plan.cpp): the
    // divisible main part of the label (its own plan sub-divides P, or splits again on the
    // other label), then the remainder accumulated into C
    std::vector<int64_t> la, lb, lta, ltb;
    const char x = p->split_label;
    int64_t len = 0;
    for (int d = 0; d < A->rank; ++d)
      if (A->labels[d] == x) len = A->lens[d];
    const tc_tensor Am = restrict_label(A, x, 0, p->split_main, esz, la);
    const tc_tensor Bm = restrict_label(B, x, 0, p->split_main, esz, lb);
    rc = tc_contract(dtype, alpha, &Am, &Bm, beta, C, stream);
    if (rc != TC_OK || len <= p->split_main) return rc;
    const tc_tensor At = restrict_label(A, x, p->split_main, len - p->split_main, esz, lta);
    const tc_tensor Bt = restrict_label(B, x, p->split_main, len - p->split_main, esz, ltb);
    return tc_contract(dtype, alpha, &At, &Bt, 1.0, C, stream);
  }
  return execute(*p, alpha, A->data, B->data, beta, C->data, static_cast<cudaStream_t>(stream));
}

int tc_contract_host(tc_dtype dtype, double alpha, const tc_tensor* A, const tc_tensor* B,
                     double beta, const tc_tensor* C, void* stream) {
  return contract_host(dtype, alpha, A, B, beta, C, static_cast<cudaStream_t>(stream));
}

int tc_release_staging(void) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  int cur = -1;
  cudaGetDevice(&cur);
  for (auto& kv : g_stage) {
    cudaSetDevice(kv.first);
    for (auto& b : kv.second.buf) { cudaFree(b); b = nullptr; }
    for (auto& c : kv.second.cap) c = 0;
  }
  if (cur >= 0) cudaSetDevice(cur);
  return TC_OK;
}

int tc_plan_create(tc_plan** plan, tc_dtype dtype, const tc_tensor* A, const tc_tensor* B,
                   const tc_tensor* C) {
  if (!plan) return fail(TC_ERR_ARG, "null plan pointer");
  int rc;
  if ((rc = check_tensor(A, "A")) || (rc = check_tensor(B, "B")) || (rc = check_tensor(C, "C")))
    return rc;
  auto* p = new (std::nothrow) Plan();
  if (!p) return fail(TC_ERR_NOMEM, "plan allocation");
  Status st = build_plan(dtype, *A, *B, *C, p);
  if (!st) { delete p; return fail(st); }
  *plan = reinterpret_cast<tc_plan*>(p);
  return TC_OK;
}

int tc_plan_execute(const tc_plan* plan, double alpha, const void* A, const void* B, double beta,
                    void* C, void* stream) {
  if (!plan) return fail(TC_ERR_ARG, "null plan");
  Nvtx range("tc_plan_execute");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  // the same alias check as tc_contract (reading R7), on the spans the plan recorded
  const int64_t esz = p.dtype == TC_F64 ? 8 : 4;
  auto bytes = [&](const void* d, int t, const char** lo, const char** hi) {
    if (!d || p.span_lo[t] > p.span_hi[t]) return false;
    *lo = static_cast<const char*>(d) + p.span_lo[t] * esz;
    *hi = static_cast<const char*>(d) + (p.span_hi[t] + 1) * esz;
    return true;
  };
  const char *c0, *c1, *x0, *x1;
  if (bytes(C, 2, &c0, &c1))
    for (int t = 0; t < 2; ++t)
      if (bytes(t == 0 ? A : B, t, &x0, &x1) && x0 < c1 && c0 < x1)
        return fail(TC_ERR_ALIAS, "C overlaps A or B");
  return execute(p, alpha, A, B, beta, C, static_cast<cudaStream_t>(stream));
}

int tc_plan_destroy(tc_plan* plan) {
  delete reinterpret_cast<Plan*>(plan);
  return TC_OK;
}

int tc_plan_query(const tc_plan* plan, tc_plan_info* info) {
  if (!plan || !info) return fail(TC_ERR_ARG, "null argument");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  info->m = p.m; info->n = p.n; info->k = p.k;
  info->flops = 2 * p.m * p.n * p.k;
  info->swapped = p.b.swapped ? 1 : 0;
  info->ndims[0] = (int32_t)p.b.I.size();
  info->ndims[1] = (int32_t)p.b.J.size();
  info->ndims[2] = (int32_t)p.b.P.size();
  info->a_vec_m = p.a_vec_m; info->b_vec_k = p.b_vec_k;
  info->idx64 = p.idx64; info->variant = p.variant;
  return TC_OK;
}

int tc_plan_dim(const tc_plan* plan, int which, int idx, int64_t* len, int64_t* s0, int64_t* s1,
                char* labels, int cap) {
  if (!plan) return fail(TC_ERR_ARG, "null plan");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  const std::vector<Dim>* b = which == 0 ? &p.b.I : which == 1 ? &p.b.J : which == 2 ? &p.b.P : nullptr;
  if (!b || idx < 0 || idx >= (int)b->size()) return fail(TC_ERR_ARG, "bad bundle/dim index");
  const Dim& d = (*b)[(size_t)idx];
  if (len) *len = d.len;
  if (s0) *s0 = d.s[0];
  if (s1) *s1 = d.s[1];
  if (labels && cap > 0) {
    std::snprintf(labels, (size_t)cap, "%s", d.labels.c_str());
  }
  return TC_OK;
}

int tc_plan_scatter(const tc_plan* plan, int which, int64_t* out, int64_t cap, int64_t* len) {
  if (!plan || which < 0 || which > 5) return fail(TC_ERR_ARG, "bad argument");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  const auto& v = p.scat[which];
  if (len) *len = (int64_t)v.size();
  if (out)
    for (int64_t i = 0; i < cap && i < (int64_t)v.size(); ++i) out[i] = v[(size_t)i];
  return TC_OK;
}

int tc_plan_traversal_scatter(const tc_plan* plan, int which, int64_t* out, int64_t cap,
                              int64_t* len) {
  if (!plan || which < 0 || which > 5) return fail(TC_ERR_ARG, "bad argument");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  const auto& v = p.kscat[which];
  if (len) *len = (int64_t)v.size();
  if (out)
    for (int64_t i = 0; i < cap && i < (int64_t)v.size(); ++i) out[i] = v[(size_t)i];
  return TC_OK;
}

int tc_plan_block_scatter(const tc_plan* plan, int which, int64_t b, int64_t* out, int64_t cap,
                          int64_t* len) {
  if (!plan || which < 0 || which > 5 || b <= 0) return fail(TC_ERR_ARG, "bad argument");
  const Plan& p = *reinterpret_cast<const Plan*>(plan);
  std::vector<int64_t> bs = block_scatter(p.scat[which], b);
  if (len) *len = (int64_t)bs.size();
  if (out)
    for (int64_t i = 0; i < cap && i < (int64_t)bs.size(); ++i) out[i] = bs[(size_t)i];
  return TC_OK;
}

const char* tc_error_string(int code) {
  switch (code) {
    case TC_OK: return "ok";
    case TC_ERR_ARG: return "invalid argument";
    case TC_ERR_LABEL: return "invalid labels";
    case TC_ERR_SHAPE: return "length mismatch";
    case TC_ERR_ALIAS: return "aliasing output";
    case TC_ERR_UNSUPPORTED: return "unsupported";
    case TC_ERR_CUDA: return "CUDA error";
    case TC_ERR_NOMEM: return "out of memory";
    default: return "unknown error";
  }
}

const char* tc_last_error_detail(void) { return g_detail.c_str(); }

int tc_version(void) { return TC_VERSION; }

}  // extern "C"
