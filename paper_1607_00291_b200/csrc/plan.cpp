// Host planner for the transposition-free contraction (steps a1-a4 of DESIGN.md §Path).
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace tcb {

static int find_label(const tc_tensor& t, char x) {
  for (int i = 0; i < t.rank; ++i)
    if (t.labels[i] == x) return i;
  return -1;
}

// a1 -- PAPER.md P:262-275: the labels of A and C form I, those of B and C form J, those of
// A and B form P; a label in one tensor or in all three, or repeated within one, is rejected
// (reading R6). Bundle order: I and P follow A's label order, J follows B's.
Status classify(const tc_tensor& A, const tc_tensor& B, const tc_tensor& C, Bundles* out) {
  const tc_tensor* T[3] = {&A, &B, &C};
  for (int t = 0; t < 3; ++t) {
    for (int i = 0; i < T[t]->rank; ++i) {
      for (int j = 0; j < i; ++j)
        if (T[t]->labels[i] == T[t]->labels[j])
          return Status::err(TC_ERR_LABEL, std::string("label '") + T[t]->labels[i] +
                                               "' repeated within one tensor");
      char x = T[t]->labels[i];
      int cnt = (find_label(A, x) >= 0) + (find_label(B, x) >= 0) + (find_label(C, x) >= 0);
      if (cnt != 2)
        return Status::err(TC_ERR_LABEL, std::string("label '") + x + "' appears in " +
                                             std::to_string(cnt) + " tensor(s), must be 2");
    }
  }
  Bundles b;
  for (int i = 0; i < A.rank; ++i) {
    char x = A.labels[i];
    int ic = find_label(C, x);
    Dim d;
    d.len = A.lens[i];
    d.labels = std::string(1, x);
    if (ic >= 0) {
      if (C.lens[ic] != d.len)
        return Status::err(TC_ERR_SHAPE, std::string("length mismatch for '") + x + "'");
      d.s[0] = A.strides[i];
      d.s[1] = C.strides[ic];
      b.I.push_back(d);
    } else {
      int ib = find_label(B, x);
      if (B.lens[ib] != d.len)
        return Status::err(TC_ERR_SHAPE, std::string("length mismatch for '") + x + "'");
      d.s[0] = A.strides[i];
      d.s[1] = B.strides[ib];
      b.P.push_back(d);
    }
  }
  for (int i = 0; i < B.rank; ++i) {
    char x = B.labels[i];
    int ic = find_label(C, x);
    if (ic < 0) continue;
    if (C.lens[ic] != B.lens[i])
      return Status::err(TC_ERR_SHAPE, std::string("length mismatch for '") + x + "'");
    Dim d;
    d.len = B.lens[i];
    d.labels = std::string(1, x);
    d.s[0] = B.strides[i];
    d.s[1] = C.strides[ic];
    b.J.push_back(d);
  }
  *out = std::move(b);
  return Status::ok();
}

// Step 2, reading R9: v folds into u when s_v = s_u * n_u in both carrying tensors;
// pairs searched u-major over the current order, repeated until no pair folds.
static void fold(std::vector<Dim>& dims) {
  for (;;) {
    bool merged = false;
    for (size_t u = 0; u < dims.size() && !merged; ++u) {
      for (size_t v = 0; v < dims.size(); ++v) {
        if (u == v) continue;
        const Dim &du = dims[u], &dv = dims[v];
        if (dv.s[0] == du.s[0] * du.len && dv.s[1] == du.s[1] * du.len) {
          dims[u].labels += dv.labels;
          dims[u].len *= dv.len;
          dims.erase(dims.begin() + (long)v);
          merged = true;
          break;
        }
      }
    }
    if (!merged) return;
  }
}

static void sort_by(std::vector<Dim>& d, int which) {
  std::stable_sort(d.begin(), d.end(), [which](const Dim& x, const Dim& y) {
    return std::llabs(x.s[which]) < std::llabs(y.s[which]);
  });
}

// a2 -- the five steps of P:926-934 in the paper's order (readings R9, R10).
void normalize(Bundles* b) {
  auto drop1 = [](std::vector<Dim>& d) {
    d.erase(std::remove_if(d.begin(), d.end(), [](const Dim& x) { return x.len == 1; }),
            d.end());
  };
  drop1(b->I); drop1(b->J); drop1(b->P);                  // 1
  fold(b->I); fold(b->J); fold(b->P);                     // 2
  sort_by(b->I, 1); sort_by(b->J, 1);                     // 3: C is stride slot 1 for I, J
  b->swapped = false;
  if (!b->J.empty() && b->J[0].s[1] == 1) {               // 4
    std::swap(b->I, b->J);                                // I now carries (B_old, C) = (A, C)
    for (auto& d : b->P) std::swap(d.s[0], d.s[1]);       // P: (A, B) after the swap
    b->swapped = true;
  }
  sort_by(b->P, 0);                                       // 5: by stride in (new) A
}

// a3 -- scat_k = sum_d digit_d(k) * s_d, digits colexicographic.
std::vector<int64_t> scatter(const std::vector<Dim>& dims, int which) {
  int64_t total = 1;
  for (const auto& d : dims) total *= d.len;
  std::vector<int64_t> out((size_t)std::max<int64_t>(total, 0));
  if (total <= 0) return out;
  // incremental odometer over the dims (same values as decoding each k)
  std::vector<int64_t> idx(dims.size(), 0);
  int64_t off = 0;
  for (int64_t k = 0; k < total; ++k) {
    out[(size_t)k] = off;
    for (size_t d = 0; d < dims.size(); ++d) {
      if (++idx[d] < dims[d].len) { off += dims[d].s[which]; break; }
      off -= (dims[d].len - 1) * dims[d].s[which];
      idx[d] = 0;
    }
  }
  return out;
}

// a4 -- P:678-683; a one-entry block has no difference to test and gets 1 (reading R11).
std::vector<int64_t> block_scatter(const std::vector<int64_t>& scat, int64_t b) {
  int64_t l = (int64_t)scat.size();
  std::vector<int64_t> out;
  if (b <= 0) return out;
  for (int64_t lo = 0; lo < l; lo += b) {
    int64_t hi = std::min(l, lo + b);
    if (hi - lo == 1) { out.push_back(1); continue; }
    int64_t s = scat[lo + 1] - scat[lo];
    bool ok = s > 0;
    for (int64_t j = lo + 1; ok && j < hi; ++j) ok = (scat[j] - scat[j - 1] == s);
    out.push_back(ok ? s : 0);
  }
  return out;
}

// Reading R7: drop length <= 1 dims, sort by |stride|, each |s| must exceed the extent
// spanned by all smaller ones.
bool injective(int rank, const int64_t* lens, const int64_t* strides) {
  std::vector<std::pair<int64_t, int64_t>> d;
  for (int i = 0; i < rank; ++i) {
    if (lens[i] == 0) return true;  // empty tensor
    if (lens[i] > 1) d.push_back({std::llabs(strides[i]), lens[i]});
  }
  std::sort(d.begin(), d.end());
  int64_t reach = 0;
  for (auto& x : d) {
    if (x.first < reach + 1) return false;
    reach += x.first * (x.second - 1);
  }
  return true;
}

void span(int rank, const int64_t* lens, const int64_t* strides, int64_t* lo, int64_t* hi) {
  int64_t a = 0, b = 0;
  for (int i = 0; i < rank; ++i) {
    if (lens[i] == 0) { *lo = 1; *hi = 0; return; }
    int64_t e = strides[i] * (lens[i] - 1);
    if (e < 0) a += e; else b += e;
  }
  *lo = a; *hi = b;
}

// True when every block of V entries of `vtab` is contiguous (block-scatter entry 1 with block
// size V), vtab's length is a multiple of V, and every block start and every entry
// of `other` is a multiple of V -- then base + vtab[V i] + other[r] (and the zero-fill
// addresses of padded rows, whose table entries are 0) is 16-byte aligned for a 16-byte
// aligned base (V = 16 / element size), and the kernel moves each block with one 16-byte copy
// without per-element checks.
// TC_KBLOCK=flat: the one-level P sub-division only (measurement A/B of the second level).
// Read per plan build (plans are cached by structure, so set it before the first call).
static bool kblock_flat() {
  const char* e = getenv("TC_KBLOCK");
  return e && !strcmp(e, "flat");
}

static bool vec_blocks_all(const std::vector<int64_t>& vtab, const std::vector<int64_t>& other,
                           int64_t V) {
  if (vtab.empty() || other.empty() || vtab.size() % (size_t)V) return false;
  for (size_t i = 0; i < vtab.size(); i += (size_t)V) {
    if (vtab[i] % V) return false;
    for (int64_t j = 1; j < V; ++j)
      if (vtab[i + (size_t)j] != vtab[i] + j) return false;
  }
  for (int64_t x : other)
    if (x % V) return false;
  return true;
}

static int64_t max_abs_offset(int rank, const int64_t* lens, const int64_t* strides) {
  int64_t s = 0;
  for (int i = 0; i < rank; ++i)
    if (lens[i] > 0) s += std::llabs(strides[i]) * (lens[i] - 1);
  return s;
}

Status build_plan(tc_dtype dtype, const tc_tensor& A, const tc_tensor& B, const tc_tensor& C,
                  Plan* p) {
  const tc_tensor* T[3] = {&A, &B, &C};
  if (dtype != TC_F64 && dtype != TC_F32) return Status::err(TC_ERR_ARG, "bad dtype");
  for (int t = 0; t < 3; ++t) {
    if (T[t]->rank < 0) return Status::err(TC_ERR_ARG, "negative rank");
    if (T[t]->rank > TC_MAX_RANK)
      return Status::err(TC_ERR_UNSUPPORTED, "rank exceeds TC_MAX_RANK");
    if (T[t]->rank > 0 && (!T[t]->lens || !T[t]->strides || !T[t]->labels))
      return Status::err(TC_ERR_ARG, "null lens/strides/labels");
    for (int i = 0; i < T[t]->rank; ++i)
      if (T[t]->lens[i] < 0) return Status::err(TC_ERR_ARG, "negative length");
  }
  Status st = classify(A, B, C, &p->b);
  if (!st) return st;
  if (!injective(C.rank, C.lens, C.strides))
    return Status::err(TC_ERR_ALIAS, "C is not injective (two index tuples share an address)");
  p->dtype = dtype;
  for (int t = 0; t < 3; ++t) span(T[t]->rank, T[t]->lens, T[t]->strides, &p->span_lo[t], &p->span_hi[t]);
  p->empty_out = false;
  for (int i = 0; i < C.rank; ++i)
    if (C.lens[i] == 0) p->empty_out = true;
  bool zero_p = false;
  for (auto& d : p->b.P)
    if (d.len == 0) zero_p = true;
  if (zero_p) p->b.P.clear();  // n_P = 0: C := beta*C, modelled as an empty product (k = 0)
  normalize(&p->b);
  auto ext = [](const std::vector<Dim>& d) {
    int64_t n = 1;
    for (auto& x : d) n *= x.len;
    return n;
  };
  p->m = ext(p->b.I);
  p->n = ext(p->b.J);
  p->k = zero_p ? 0 : ext(p->b.P);
  if (p->empty_out) { p->m = 0; p->n = 0; }
  // 64-bit offsets only when some tensor spans 2^31 elements or more
  int64_t big = std::max({max_abs_offset(A.rank, A.lens, A.strides),
                          max_abs_offset(B.rank, B.lens, B.strides),
                          max_abs_offset(C.rank, C.lens, C.strides)});
  p->idx64 = big >= (int64_t(1) << 31) - 1;
  if (p->m >= (int64_t(1) << 31) || p->n >= (int64_t(1) << 31) || p->k >= (int64_t(1) << 31))
    return Status::err(TC_ERR_UNSUPPORTED, "a bundle extent exceeds 2^31");
  if (!p->empty_out) {
    p->scat[0] = scatter(p->b.I, 0);  // rscat_A
    p->scat[1] = scatter(p->b.P, 0);  // cscat_A
    p->scat[2] = scatter(p->b.P, 1);  // rscat_B
    p->scat[3] = scatter(p->b.J, 0);  // cscat_B
    p->scat[4] = scatter(p->b.I, 1);  // rscat_C
    p->scat[5] = scatter(p->b.J, 1);  // cscat_C
    if (p->k == 0) { p->scat[1].clear(); p->scat[2].clear(); }
  }
  // GPU traversal order (DESIGN.md §3 R16; "the optimal ordering ... may differ
  // from that achieved by the above heuristics"). The heuristic favours C's unit stride (sort
  // by C stride) and A's only within P. On the GPU the kernel reads A once per N tile and B once
  // per M tile, while C is written once (a partial-sector write costs about twice a read), so
  // each bundle is walked with the unit-stride dimension of the tensor that moves the most
  // elements through it first: in I, A's (weight K*M*ceil(N/128)) against C's (2*M*N); in P,
  // A's, or B's when A took I; in J, B's (K*N*ceil(M/128)) against C's, when B did not take P.
  // Values are unchanged (same elements, other tile membership); the paper-order tables above
  // stay the plan's reported scatter vectors.
  p->kb = p->b;
  auto find_unit = [](const std::vector<Dim>& d, int w) {
    for (size_t i = 0; i < d.size(); ++i)
      if (d[i].s[w] == 1) return (int)i;
    return -1;
  };
  auto to_front = [](std::vector<Dim>& d, int i) {
    if (i > 0) { Dim x = d[(size_t)i]; d.erase(d.begin() + i); d.insert(d.begin(), x); }
  };
  auto unit_front = [&](std::vector<Dim>& d, int w) {
    const int i = find_unit(d, w);
    to_front(d, i);
    return i >= 0;
  };
  const double tiles_n = (double)((p->n + kTileN - 1) / kTileN);
  const double tiles_m = (double)((p->m + kTileM - 1) / kTileM);
  const double wA = (double)p->k * (double)p->m * tiles_n;
  const double wB = (double)p->k * (double)p->n * tiles_m;
  const double wC = 2.0 * (double)p->m * (double)p->n;
  bool a_m = false;
  {
    const int ia = find_unit(p->kb.I, 0), ic = find_unit(p->kb.I, 1);
    if (ia >= 0 && (ic < 0 || ic == ia || wA > wC)) { to_front(p->kb.I, ia); a_m = true; }
    else to_front(p->kb.I, ic);
  }
  // Dimension sub-division of P: when A and B both read along
  // K but have different unit-stride dimensions u (A's) and w (B's) there, the bundle is walked
  // as [u_lo, w_lo, u_hi, w_hi, rest] with u_lo, w_lo of length <= 4 (powers of two dividing
  // the lengths), so within each K step both operands read runs of consecutive elements
  // instead of one of them gathering element by element.
  p->k_blocked = false;
  if (!a_m && p->k > 0) {
    const int u = find_unit(p->kb.P, 0), w = find_unit(p->kb.P, 1);
    auto divisor = [](int64_t len) {
      for (int64_t b = 4; b >= 2; b /= 2)
        if (len % b == 0) return b;
      return (int64_t)1;
    };
    if (u >= 0 && w >= 0 && u != w) {
      const Dim du = p->kb.P[(size_t)u], dw = p->kb.P[(size_t)w];
      const int64_t bu = divisor(du.len), bw = divisor(dw.len);
      if (bu > 1 && bw > 1) {
        auto part = [](const Dim& d, int64_t len, int64_t mul, const char* tag) {
          Dim x = d;
          x.len = len;
          x.s[0] = d.s[0] * mul;
          x.s[1] = d.s[1] * mul;
          x.labels = d.labels + tag;
          return x;
        };
        std::vector<Dim> out = {part(du, bu, 1, "_lo"), part(dw, bw, 1, "_lo")};
        // Second level when both lengths allow it (bu = bw = 4, both lengths multiples of 16):
        // [u_lo, w_lo, u_mid, w_mid, u_hi, w_hi], so every 16 consecutive K steps read whole
        // 128-byte lines of both operands (u 0..15 x w 0..15) instead of 32-byte pieces whose
        // line-mates come back 1/4 of the bundle later (fig:bench ab-cad-dcb: 3.6 GB of DRAM
        // reads for 0.54 GB of operands, profiles/r02/ncu/f2_16_k2.summary.txt)
        const bool mid = bu == 4 && bw == 4 && du.len % 16 == 0 && dw.len % 16 == 0 &&
                         du.len > 16 && dw.len > 16 && !kblock_flat();
        if (mid) {
          out.push_back(part(du, 4, 4, "_mid"));
          out.push_back(part(dw, 4, 4, "_mid"));
          out.push_back(part(du, du.len / 16, 16, "_hi"));
          out.push_back(part(dw, dw.len / 16, 16, "_hi"));
        } else {
          if (du.len / bu > 1) out.push_back(part(du, du.len / bu, bu, "_hi"));
          if (dw.len / bw > 1) out.push_back(part(dw, dw.len / bw, bw, "_hi"));
        }
        for (size_t i = 0; i < p->kb.P.size(); ++i)
          if ((int)i != u && (int)i != w) out.push_back(p->kb.P[i]);
        p->kb.P = out;
        p->k_blocked = true;
      } else {
        // A length with no divisor <= 4 (e.g. 323 = 17 * 19, fig:bench's ab-cad-dcb): if it is a
        // single label and both dimensions are long, record a split of that label at the
        // largest multiple of 4; the device entry point runs the divisible main part (which is
        // then sub-divided) and the small remainder as separate contractions
        const Dim& dx = bu == 1 ? du : dw;
        const Dim& dy = bu == 1 ? dw : du;
        if (dx.labels.size() == 1 && dx.len >= 64 && dy.len >= 64) {
          p->split_label = dx.labels[0];
          p->split_main = dx.len - dx.len % 4;
        }
      }
    }
  }
  bool a_k = !a_m && (p->k_blocked || unit_front(p->kb.P, 0));
  bool b_k = p->k_blocked ||
             (a_k ? (!p->kb.P.empty() && p->kb.P[0].s[1] == 1) : unit_front(p->kb.P, 1));
  if (!b_k) {
    const int jb = find_unit(p->kb.J, 0), jc = find_unit(p->kb.J, 1);
    if (jb >= 0 && (jc < 0 || jc == jb || wB > wC)) to_front(p->kb.J, jb);
    else to_front(p->kb.J, jc);
  }
  // Dimension sub-division for skinny contractions (the paper's remedy for
  // contractions without a common stride-1 index). When the skinny kernel will
  // stream the long free bundle (fp64, K <= 80, the other free extent <= 96) and the streamed
  // operand X and C have different unit-stride dimensions u (X's) and v (C's) in it, the bundle
  // is walked as [v_lo, u_lo, u_hi, v_hi, rest] with v_lo, u_lo the largest divisors of the two
  // lengths that are <= 8: a block of rows then holds bv runs of bu consecutive X elements and
  // bu runs of bv consecutive C elements, so both streams move whole sectors. The kernel's
  // loader maps lanes to rows through (bu, bv).
  p->skinny_bu = p->skinny_bv = 1;
  if (dtype == TC_F64 && !p->empty_out && p->k >= 1 && p->k <= 80 &&
      (p->n <= 96 || p->m <= 96)) {
    std::vector<Dim>& L = p->n <= 96 ? p->kb.I : p->kb.J;   // long bundle; X = A or B
    const int u = find_unit(L, 0), v = find_unit(L, 1);
    auto divisor = [](int64_t len, int64_t cap) {   // a power of two, so bu * bv divides the
      for (int64_t b = cap; b >= 2; b /= 2)           // 64-row block
        if (len % b == 0) return b;
      return (int64_t)1;
    };
    // run-length caps (measurement overrides read per plan): TC_SKINNY_BV = 2..32 for C's runs,
    // TC_SKINNY_BU = 2..32 for X's; the other then caps at 64 / that one (measured: 8 and 8,
    // profiles/r02/ab_skinny_runs.txt)
    auto cap_env = [](const char* name) -> int64_t {
      const char* e = getenv(name);
      const int64_t c = e ? atoi(e) : 0;
      return c == 2 || c == 4 || c == 8 || c == 16 || c == 32 ? c : 0;
    };
    const int64_t bv_env = cap_env("TC_SKINNY_BV"), bu_env = cap_env("TC_SKINNY_BU");
    if (u >= 0 && v >= 0 && u != v) {
      int64_t bv, bu;
      if (bu_env) {
        bu = divisor(L[(size_t)u].len, bu_env);
        bv = divisor(L[(size_t)v].len, std::min<int64_t>(bv_env ? bv_env : 8, 64 / bu));
      } else {
        bv = divisor(L[(size_t)v].len, bv_env ? bv_env : 8);
        bu = divisor(L[(size_t)u].len, std::min<int64_t>(8, 64 / bv));
      }
      if (bu > 1 && bv > 1) {
        const Dim du = L[(size_t)u], dv = L[(size_t)v];
        auto part = [](const Dim& d, int64_t len, int64_t mul, const char* tag) {
          Dim x = d;
          x.len = len;
          x.s[0] = d.s[0] * mul;
          x.s[1] = d.s[1] * mul;
          x.labels = d.labels + tag;
          return x;
        };
        std::vector<Dim> out = {part(dv, bv, 1, "_lo"), part(du, bu, 1, "_lo")};
        if (du.len / bu > 1) out.push_back(part(du, du.len / bu, bu, "_hi"));
        if (dv.len / bv > 1) out.push_back(part(dv, dv.len / bv, bv, "_hi"));
        for (size_t i = 0; i < L.size(); ++i)
          if ((int)i != u && (int)i != v) out.push_back(L[i]);
        L = out;
        p->skinny_bu = (int)bu;
        p->skinny_bv = (int)bv;
      }
    }
  }
  if (!p->empty_out) {
    p->kscat[0] = scatter(p->kb.I, 0);
    p->kscat[1] = scatter(p->kb.P, 0);
    p->kscat[2] = scatter(p->kb.P, 1);
    p->kscat[3] = scatter(p->kb.J, 0);
    p->kscat[4] = scatter(p->kb.I, 1);
    p->kscat[5] = scatter(p->kb.J, 1);
    if (p->k == 0) { p->kscat[1].clear(); p->kscat[2].clear(); }
  }
  // Loader direction per operand: gather along the bundle whose first dimension has unit
  // stride (16-byte vectors, coalesced warps); else along the smaller leading stride.
  auto lead = [](const std::vector<Dim>& d, int w) {
    return d.empty() ? INT64_MAX : std::llabs(d[0].s[w]);
  };
  int64_t la_m = lead(p->kb.I, 0), la_k = lead(p->kb.P, 0);
  int64_t lb_k = lead(p->kb.P, 1), lb_n = lead(p->kb.J, 0);
  p->a_vec_m = la_m <= la_k;
  p->b_vec_k = lb_k <= lb_n;
  if (p->k_blocked) {   // both operands read their runs along the sub-divided K
    p->a_vec_m = false;
    p->b_vec_k = true;
  }
  if (p->skinny_bu > 1) {   // the sub-divided long bundle is the streamed operand's direction
    if (p->n <= 96) p->a_vec_m = true;
    else p->b_vec_k = false;
  }
  if (!p->empty_out && p->k > 0) {
    const int64_t V = dtype == TC_F64 ? 2 : 4;
    p->a_pairs_all = p->a_vec_m ? vec_blocks_all(p->kscat[0], p->kscat[1], V)
                                : vec_blocks_all(p->kscat[1], p->kscat[0], V);
    p->b_pairs_all = p->b_vec_k ? vec_blocks_all(p->kscat[2], p->kscat[3], V)
                                : vec_blocks_all(p->kscat[3], p->kscat[2], V);
    if (dtype == TC_F32) {
      p->a_pairs2_all = p->a_vec_m ? vec_blocks_all(p->kscat[0], p->kscat[1], 2)
                                   : vec_blocks_all(p->kscat[1], p->kscat[0], 2);
      p->b_pairs2_all = p->b_vec_k ? vec_blocks_all(p->kscat[2], p->kscat[3], 2)
                                   : vec_blocks_all(p->kscat[3], p->kscat[2], 2);
    }
  }
  // Gather mode of an operand that is not all-vector (contract_ws.cuh GatherSel), measured on
  // the cfg4 / f2 suites (profiles/r01/suite_gather_ab.txt): for fp32 the coalesced element
  // gather wins (a 16-byte vector holds 4 elements, so odd runs misalign most vectors); for fp64
  // the per-vector check is as good or better (2-element vectors are mostly aligned).
  p->a_elem = p->b_elem = dtype == TC_F32;

  auto unit_steps = [](const std::vector<int64_t>& t) {
    int64_t u = 0;
    for (size_t i = 1; i < t.size(); ++i) u += t[i] - t[i - 1] == 1;
    return (double)u / (double)(t.size() > 1 ? t.size() - 1 : 1);
  };
  if (!p->empty_out) p->c_unit_n = unit_steps(p->kscat[5]) > unit_steps(p->kscat[4]);
  p->variant = (p->a_vec_m ? 1 : 0) | (p->b_vec_k ? 2 : 0) | (p->idx64 ? 4 : 0) |
               (dtype == TC_F32 ? 8 : 0) |
               (p->c_unit_n ? 16 : 0);
  return Status::ok();
}

}  // namespace tcb
