// Host-side planner: index bundles, the section 7.3 heuristic, scatter and block-scatter
// vectors, kernel-variant selection. Pure C++17, no CUDA; the device side lives in
// contract_kernels.cu and tc_api.cpp uploads the tables.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "tc.h"

namespace tcb {

// One (possibly folded) dimension of a bundle. s[0], s[1] are its strides in the two tensors
// carrying the bundle: I -> (A, C), J -> (B, C), P -> (A, B), in the roles after the swap.
struct Dim {
  int64_t len = 1;
  int64_t s[2] = {0, 0};
  std::string labels;  // original labels, fastest first
};

struct Bundles {
  std::vector<Dim> I, J, P;
  bool swapped = false;
};

struct Status {
  int code = TC_OK;
  std::string detail;
  static Status ok() { return {}; }
  static Status err(int c, std::string d) { return {c, std::move(d)}; }
  explicit operator bool() const { return code == TC_OK; }
};

// a1: classify labels into I (A and C), J (B and C), P (A and B) -- PAPER.md P:262-298.
Status classify(const tc_tensor& A, const tc_tensor& B, const tc_tensor& C, Bundles* out);

// a2: the heuristic of P:926-934 (drop length-1 dims, fold sequentially contiguous dims, sort
// I/J by C stride, swap if s_{j0}(C) == 1, sort P by A stride).
void normalize(Bundles* b);

// a3: scatter vector of a bundle in one tensor (generic P:577-579).
std::vector<int64_t> scatter(const std::vector<Dim>& dims, int which_stride);

// a4: block-scatter vector with block size b.
std::vector<int64_t> block_scatter(const std::vector<int64_t>& scat, int64_t b);

// Injectivity of a strided layout (sufficient test, reading R7).
bool injective(int rank, const int64_t* lens, const int64_t* strides);

// [lo, hi] element-offset span of a strided tensor (empty tensors: lo > hi).
void span(int rank, const int64_t* lens, const int64_t* strides, int64_t* lo, int64_t* hi);

// CTA tile of the contraction kernel (kernels.hpp kBM, kBN), for the traversal-order cost model
constexpr int64_t kTileM = 128, kTileN = 128;

struct DeviceTables;  // defined in tc_api.cpp

struct Plan {
  tc_dtype dtype = TC_F64;
  Bundles b;
  int64_t m = 1, n = 1, k = 1;
  bool empty_out = false;  // some free length is 0: no-op
  // scatter vectors, roles after the swap: 0 rA, 1 cA, 2 rB, 3 cB, 4 rC, 5 cC
  std::vector<int64_t> scat[6];
  // GPU traversal order of the bundles (unit-stride dimensions of A, B first) and the scatter
  // vectors the kernel walks (same elements, other linearisation)
  Bundles kb;
  std::vector<int64_t> kscat[6];
  bool a_vec_m = true;     // loader direction of A (true: along M)
  bool b_vec_k = true;     // loader direction of B (true: along K)
  bool idx64 = false;
  // whole-operand block-scatter check at 16-byte granularity (see vec_blocks_all in plan.cpp)
  bool a_pairs_all = false, b_pairs_all = false;
  // the same at 8-byte granularity (fp32: pairs of floats), for the tcgen05 kernel's 8-byte gathers
  bool a_pairs2_all = false, b_pairs2_all = false;
  // gather mode for operands that are not all-vector: coalesced element copies (true) or the
  // per-vector check (false), from the share of vectors that qualify (plan.cpp)
  bool a_elem = true, b_elem = true;
  // C's traversal tables: more unit steps along N (cscat_C) than along M (rscat_C)
  bool c_unit_n = false;
  // row blocking of the long free bundle for the skinny kernel (1, 1: none), see plan.cpp
  int skinny_bu = 1, skinny_bv = 1;
  bool k_blocked = false;   // P walked as [u_lo, w_lo, u_hi, w_hi, ...] (plan.cpp)
  // sub-division blocked by a length without a small power-of-two divisor (plan.cpp): the
  // contraction is run as a main part over split_label in [0, split_main), which can be
  // sub-divided, plus the remainder (tc_api.cpp); 0 = no split
  char split_label = 0;
  int64_t split_main = 0;
  int variant = 0;
  // element-offset spans [lo, hi] of A, B, C (caller's roles, before any swap): the alias
  // check of tc_plan_execute, which gets bare data pointers
  int64_t span_lo[3] = {1, 1, 1}, span_hi[3] = {0, 0, 0};
  // per-device uploaded tables
  mutable std::mutex mu;
  mutable std::vector<DeviceTables*> dev;
  ~Plan();
};

Status build_plan(tc_dtype dtype, const tc_tensor& A, const tc_tensor& B, const tc_tensor& C,
                  Plan* p);

}  // namespace tcb
