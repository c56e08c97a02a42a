/*
 * tc.h -- C ABI of the B200 (sm_100a) transposition-free tensor contraction library
 *         (libtc_b200.so, built from paper_1607_00291_b200/csrc/).
 *
 * The operation (§4, Eq. P:278-281 / eq:gen-contraction P:296-298, with alpha and beta
 * from P:193):
 *
 *     C[pi_C(I J)] := alpha * sum_P A[pi_A(I P)] * B[pi_B(P J)] + beta * C[pi_C(I J)]
 *
 * over tensors of any rank (<= TC_MAX_RANK) and any element strides (loc = sum idx*stride,
 * P:563-571). Labels name the indices: a label in A and C is free (bundle I), in B and C free
 * (bundle J), in A and B bound (bundle P, summed); every label must occur in exactly two of the
 * three tensors, once. The index permutation is folded into the kernel's tile loads
 * through scatter / block-scatter vectors (§6); no operand is transposed and no
 * operand-sized workspace is allocated.
 *
 * Conventions for every entry point:
 *   - dtype: all three tensors share one element type (TC_F64 or TC_F32).
 *   - lens[i] >= 0 are element counts; strides[i] are signed element (not byte) strides.
 *   - labels: exactly `rank` bytes (not necessarily NUL-terminated), no repeats in one tensor.
 *   - data: pointer to element (0,...,0) -- DEVICE memory for tc_contract / tc_plan_execute,
 *     HOST memory for tc_contract_host. It must be aligned to the element size.
 *   - Host arrays (lens, strides, labels) are read during the call only; nothing is retained.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Semantics (readings R1, R8): beta == 0 => C is write-only (never read, so NaN in
 *     C is harmless); alpha == 0 => A and B are not read; a zero-length free index => no-op;
 *     a zero-length bound index => C := beta*C; an empty bundle has extent 1 (d_P = 0 is an
 *     outer product; d_I = d_J = 0 writes a scalar).
 *   - C must be injective (no two index tuples at one address, "preserves the
 *     uniqueness of elements") and must not overlap A or B; A and B may use zero strides.
 *   - Return value: TC_OK or a TC_ERR_* code; validation errors return before anything is
 *     enqueued. tc_last_error_detail() gives a thread-local message for the last failure.
 * Thread safety: all entry points may be called concurrently; the internal plan cache is locked.
 */
#ifndef TC_B200_H
#define TC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_MAX_RANK 16
#define TC_VERSION 100

typedef enum { TC_F64 = 0, TC_F32 = 1 } tc_dtype;

enum {
  TC_OK = 0,
  TC_ERR_ARG = 1,          /* null pointer, bad rank, bad dtype, misaligned data           */
  TC_ERR_LABEL = 2,        /* label in 1 or 3 tensors, or repeated in one       */
  TC_ERR_SHAPE = 3,        /* a shared label with different lengths            */
  TC_ERR_ALIAS = 4,        /* C not injective, or C overlaps A or B                         */
  TC_ERR_UNSUPPORTED = 5,  /* rank > TC_MAX_RANK, extents beyond the kernel's index range   */
  TC_ERR_CUDA = 6,         /* CUDA runtime / launch error (detail string set)               */
  TC_ERR_NOMEM = 7         /* host or device allocation failure                             */
};

/* One strided tensor operand (SPEC.md S:31-37 DenseTensor). */
typedef struct {
  int32_t rank;            /* 0..TC_MAX_RANK                                                */
  const int64_t* lens;     /* [rank] lengths, >= 0                                          */
  const int64_t* strides;  /* [rank] signed element strides                                 */
  const char* labels;      /* [rank] single-byte index labels                               */
  void* data;              /* element (0,...,0); device or host memory per entry point      */
} tc_tensor;

/* A planned contraction: bundles, the section 7.3 heuristic, scatter and block-scatter tables
 * (built on the host; uploaded to a device on first execution there) and the kernel variant. */
typedef struct tc_plan tc_plan;

/* C := alpha*A.B + beta*C on DEVICE buffers, asynchronously on `stream`. Plans are cached by
 * (dtype, labels, lens, strides, device), so repeated calls with the same structure skip
 * planning and table upload. When the plan's P sub-division is blocked by a long bound length
 * with no small power-of-two divisor (R17), the call runs as two or more kernel
 * launches on `stream`: the divisible main part of that label (with beta), then the remainder
 * accumulated into C (beta = 1); the result is the same contraction. */
int tc_contract(tc_dtype dtype, double alpha, const tc_tensor* A, const tc_tensor* B,
                double beta, const tc_tensor* C, void* stream);

/* Same operation on HOST buffers (the end-to-end path). Copies the address spans of A and B
 * (and of C when beta != 0, or when C's span has holes) to device staging memory, contracts,
 * copies C's span back, and synchronises `stream` before returning. The work is cut into up
 * to 8 chunks along one free label x of C (the one with C's largest stride whose chunks are
 * disjoint address intervals and which adds at most 5% copy volume), so host->device copies,
 * kernels and device->host copies of consecutive chunks overlap on three streams. The operand
 * without x (needed by every chunk) is uploaded first, or, when it has a bound label whose
 * chunks are contiguous, streamed in up to 8 pieces behind the first chunk's kernels (that
 * chunk is then summed over the pieces: beta on the first, 1 after). Otherwise one chunk.
 * Pinned host memory gives full copy bandwidth and overlap; pageable memory works. Elements of
 * C's span that are not elements of C are preserved. The staging memory (the spans of A, B, C)
 * is kept per device between calls; tc_release_staging() frees it. Calls on one device are
 * serialised by an internal lock. */
int tc_contract_host(tc_dtype dtype, double alpha, const tc_tensor* A, const tc_tensor* B,
                     double beta, const tc_tensor* C, void* stream);

/* Free the device staging memory tc_contract_host keeps (all devices). Returns TC_OK. */
int tc_release_staging(void);

/* Plan from shapes/strides/labels only (the `data` fields are ignored). Host-only: needs no GPU.
 * On success *plan owns its tables; release with tc_plan_destroy. */
int tc_plan_create(tc_plan** plan, tc_dtype dtype, const tc_tensor* A, const tc_tensor* B,
                   const tc_tensor* C);

/* Execute a plan on device buffers whose structure equals the planned one (one launch, the
 * plan as built: no remainder split, see tc_contract -- the result is the same, only the
 * R17 speed-up of labels without a small power-of-two divisor is missing). The data pointers
 * are checked like tc_contract's: TC_ERR_ARG if misaligned or NULL where read, TC_ERR_ALIAS if
 * C's address span (from the planned lengths and strides) overlaps A's or B's; nothing is
 * enqueued then. */
int tc_plan_execute(const tc_plan* plan, double alpha, const void* A, const void* B,
                    double beta, void* C, void* stream);

int tc_plan_destroy(tc_plan* plan);

/* ---- introspection (host-only; used by the parity tests of steps a1-a4) ------------------- */

typedef struct {
  int64_t m, n, k;         /* extents of the folded bundles I, J, P (n_I, n_J, n_P)          */
  int64_t flops;           /* 2*m*n*k                                            */
  int32_t swapped;         /* 1 if heuristic step 4 swapped A<->B and I<->J      */
  int32_t ndims[3];        /* folded dimensions in I, J, P after the heuristic               */
  int32_t a_vec_m;         /* loader direction for A: 1 = along M (I), 0 = along K (P)       */
  int32_t b_vec_k;         /* loader direction for B: 1 = along K (P), 0 = along N (J)       */
  int32_t idx64;           /* 1 if 64-bit offsets are needed, 0 for 32-bit                   */
  int32_t variant;         /* bits: 1 A along M, 2 B along K, 4 int64 offsets, 8 fp32,       */
                           /* 16 C unit stride along N (epilogue lanes take columns)        */
} tc_plan_info;

int tc_plan_query(const tc_plan* plan, tc_plan_info* info);

/* Folded dimension `idx` of bundle `which` (0 = I, 1 = J, 2 = P) after the heuristic:
 * its length, its stride in the two tensors carrying the bundle (I: A then C; J: B then C;
 * P: A then B; A/B in the roles after the swap) and its original labels (NUL-terminated,
 * fastest first; cap >= TC_MAX_RANK + 1). */
int tc_plan_dim(const tc_plan* plan, int which, int idx, int64_t* len, int64_t* stride_first,
                int64_t* stride_second, char* labels, int cap);

/* The six scatter vectors: which = 0 rscat_A[m], 1 cscat_A[k], 2 rscat_B[k],
 * 3 cscat_B[n], 4 rscat_C[m], 5 cscat_C[n]. Copies min(cap, length) entries to out (host);
 * returns the length through *len. */
int tc_plan_scatter(const tc_plan* plan, int which, int64_t* out, int64_t cap, int64_t* len);

/* The scatter vectors the kernel actually walks (reading R16): the same six tables
 * for the GPU traversal order of each bundle, which puts A's and then B's unit-stride dimension
 * first. Same contraction, other linearisation; same arguments as tc_plan_scatter. */
int tc_plan_traversal_scatter(const tc_plan* plan, int which, int64_t* out, int64_t cap,
                              int64_t* len);

/* Block-scatter vector of scatter vector `which` with block size b: entry i is the
 * common difference s > 0 of block i, else 0 (a one-entry block gives 1). */
int tc_plan_block_scatter(const tc_plan* plan, int which, int64_t b, int64_t* out, int64_t cap,
                          int64_t* len);

const char* tc_error_string(int code);
const char* tc_last_error_detail(void);
int tc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TC_B200_H */
