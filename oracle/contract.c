/*
 * oracle/contract.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU definition of a general dense tensor contraction,
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * Nothing in the product path (paper_1607_00291_b200/, include/) may link, import or call it,
 * and it shares no code with that path.
 *
 * What it computes (§4, Eq. at P:278-281 and eq:gen-contraction P:296-298; alpha/beta
 * from P:193 and P:199; generic strided location from P:569-571):
 *
 *   C[pi_C(I J)] := alpha * sum_{P} A[pi_A(I P)] * B[pi_B(P J)] + beta * C[pi_C(I J)]
 *
 * for every free multi-index (I, J) of C, with loc(T_{u...}) = sum_x idx_x * stride_x(T).
 * Readings: R1 beta == 0 => C is not read; alpha == 0 => A, B not read;
 * R2 the sum bound of fig:TTDT is read as 0..n_P-1 (as P:199); R5 the P
 * multi-index is visited in ascending colexicographic order of the P labels as they appear
 * in A; the accumulator is double (also for float inputs, which round once at the end).
 * Compile with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Labels: each label (a byte) appears in exactly two of the three tensors;
 * otherwise the call returns a nonzero error code (R6). Lengths of a shared label must agree.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXR 32

typedef struct {
  int n;                     /* number of labels in this group */
  int64_t len[OR_MAXR];
  int64_t sa[OR_MAXR];       /* stride in A (0 if absent) */
  int64_t sb[OR_MAXR];       /* stride in B (0 if absent) */
  int64_t sc[OR_MAXR];       /* stride in C (0 if absent) */
} or_group;

static int find(const char* lab, int r, char x) {
  for (int i = 0; i < r; ++i) if (lab[i] == x) return i;
  return -1;
}

/* Classify labels into the free group F (labels of C, in C's order: I and J together) and
 * the bound group P (labels of A not in C, in A's order). Returns 0 or an error code. */
static int classify(int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                    int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                    int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                    or_group* F, or_group* P) {
  if (rA > OR_MAXR || rB > OR_MAXR || rC > OR_MAXR) return 1;
  F->n = 0; P->n = 0;
  for (int i = 0; i < rC; ++i) {           /* each C label: exactly one of A, B */
    int ia = find(labA, rA, labC[i]), ib = find(labB, rB, labC[i]);
    if (find(labC, i, labC[i]) >= 0) return 2;          /* repeated in C */
    if ((ia >= 0) == (ib >= 0)) return 2;               /* in none or in all three */
    int64_t n = lC[i];
    if (ia >= 0 && lA[ia] != n) return 3;
    if (ib >= 0 && lB[ib] != n) return 3;
    F->len[F->n] = n; F->sc[F->n] = sC[i];
    F->sa[F->n] = ia >= 0 ? sA[ia] : 0; F->sb[F->n] = ib >= 0 ? sB[ib] : 0;
    F->n++;
  }
  for (int i = 0; i < rA; ++i) {           /* A labels not in C: bound, must be in B */
    if (find(labA, i, labA[i]) >= 0) return 2;
    if (find(labC, rC, labA[i]) >= 0) continue;
    int ib = find(labB, rB, labA[i]);
    if (ib < 0) return 2;
    if (lB[ib] != lA[i]) return 3;
    P->len[P->n] = lA[i]; P->sa[P->n] = sA[i]; P->sb[P->n] = sB[ib]; P->sc[P->n] = 0;
    P->n++;
  }
  for (int i = 0; i < rB; ++i) {           /* every B label must be in A or C (once) */
    if (find(labB, i, labB[i]) >= 0) return 2;
    if (find(labA, rA, labB[i]) < 0 && find(labC, rC, labB[i]) < 0) return 2;
  }
  return 0;
}

static int64_t extent(const or_group* g) {
  int64_t n = 1;
  for (int i = 0; i < g->n; ++i) n *= g->len[i];
  return n;
}

/* Decode linear index q colexicographically over group g (first index fastest)
 * and return the location sums for A, B and C. */
static void decode(const or_group* g, int64_t q, int64_t* oa, int64_t* ob, int64_t* oc) {
  int64_t a = 0, b = 0, c = 0;
  for (int i = 0; i < g->n; ++i) {
    int64_t x = q % g->len[i];
    q /= g->len[i];
    a += x * g->sa[i]; b += x * g->sb[i]; c += x * g->sc[i];
  }
  *oa = a; *ob = b; *oc = c;
}

/* sum_P A*B for the free element whose A/B location partial sums are fa, fb. */
static double dot_f64(const double* A, const double* B, const or_group* P, int64_t nP,
                      int64_t fa, int64_t fb) {
  double s = 0.0;
  for (int64_t p = 0; p < nP; ++p) {
    int64_t pa, pb, pc;
    decode(P, p, &pa, &pb, &pc);
    s += A[fa + pa] * B[fb + pb];
  }
  return s;
}

static double dot_f32(const float* A, const float* B, const or_group* P, int64_t nP,
                      int64_t fa, int64_t fb) {
  double s = 0.0;
  for (int64_t p = 0; p < nP; ++p) {
    int64_t pa, pb, pc;
    decode(P, p, &pa, &pb, &pc);
    s += (double)A[fa + pa] * (double)B[fb + pb];
  }
  return s;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Full contraction, in place on C. dtype: 0 = double, 1 = float. */
int oracle_contract(int dtype, double alpha,
                    const void* A, int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                    const void* B, int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                    double beta,
                    void* C, int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                    int nthreads) {
  or_group F, P;
  int err = classify(rA, lA, sA, labA, rB, lB, sB, labB, rC, lC, sC, labC, &F, &P);
  if (err) return err;
  int64_t nF = extent(&F), nP = extent(&P);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < nF; ++q) {
    int64_t fa, fb, fc;
    decode(&F, q, &fa, &fb, &fc);
    double s = 0.0;
    if (alpha != 0.0)
      s = dtype == 0 ? dot_f64((const double*)A, (const double*)B, &P, nP, fa, fb)
                     : dot_f32((const float*)A, (const float*)B, &P, nP, fa, fb);
    if (dtype == 0) {
      double* c = (double*)C + fc;
      *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
    } else {
      float* c = (float*)C + fc;
      *c = (float)(beta == 0.0 ? alpha * s : alpha * s + beta * (double)*c);
    }
  }
  return 0;
}

/* Selected elements only: for each of the nsamp multi-indices of C (row-major array
 * idx[nsamp][rC], in C's label order) write alpha*sum + beta*C_old to out[] (double),
 * without modifying C. Used for full-size sampled parity. */
int oracle_contract_at(int dtype, double alpha,
                       const void* A, int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                       const void* B, int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                       double beta,
                       const void* C, int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                       int64_t nsamp, const int64_t* idx, double* out, int nthreads) {
  or_group F, P;
  int err = classify(rA, lA, sA, labA, rB, lB, sB, labB, rC, lC, sC, labC, &F, &P);
  if (err) return err;
  int64_t nP = extent(&P);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < nsamp; ++t) {
    int64_t fa = 0, fb = 0, fc = 0;
    for (int i = 0; i < rC; ++i) {
      int64_t x = idx[t * rC + i];
      fa += x * F.sa[i]; fb += x * F.sb[i]; fc += x * F.sc[i];
    }
    double s = 0.0;
    if (alpha != 0.0)
      s = dtype == 0 ? dot_f64((const double*)A, (const double*)B, &P, nP, fa, fb)
                     : dot_f32((const float*)A, (const float*)B, &P, nP, fa, fb);
    double cold = 0.0;
    if (beta != 0.0) cold = dtype == 0 ? ((const double*)C)[fc] : (double)((const float*)C)[fc];
    out[t] = beta == 0.0 ? alpha * s : alpha * s + beta * cold;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Pin p8: Freivalds' full-tensor check, for results the element-wise
 * definition above cannot finish at full size (cfg3, cfg5, each multi-GPU shard).
 *
 * View the contraction in its matrix form (§3, §6.1: every free index of
 * C is a pair (I, J), every element of A a pair (I, P), of B a pair (P, J)):
 *     C_new = alpha * A B + beta * C_old.
 * Multiplying both sides by a vector x over J (colexicographic over the J labels in C's label
 * order, the first fastest, as P:528-529) gives, for every I,
 *     sum_J C_new[I,J] x[J]  ==  alpha * sum_P A[I,P] * (sum_J B[P,J] x[J])
 *                                + beta * sum_J C_old[I,J] x[J].
 * A wrong C_new[I,J] changes the left side at I by (error * x[J]); Freivalds (1977).
 *
 * Groups: I = labels of C that are in A (C's order), J = labels of C that are in B (C's order),
 * P = labels of A not in C (A's order). Every location is loc = sum_x idx_x * stride_x
 * (P:569-571); the sum over a label group splits into the I, J, P parts, and each part is
 * tabulated once per group (offI/offJ/offP below) -- only the associativity of that sum.
 *
 * Outputs (all double, the caller owns them):
 *   u[nP]    = sum_J B[P,J] x[J]
 *   v[nI]    = sum_P A[I,P] u[P]
 *   wnew[nI] = sum_J C_new[I,J] x[J]
 *   wold[nI] = sum_J C_old[I,J] x[J]   (not computed, left untouched, when Cold == NULL)
 * Each output element is summed in ascending order of its summation index. The loops over the
 * output index are grouped in blocks of FV_BLK consecutive outputs so that consecutive output
 * elements read neighbouring memory; this changes no value (each output keeps its own
 * accumulator and its own ascending summation order).
 * Returns 0 or the same error codes as oracle_contract.
 * ---------------------------------------------------------------------------------------- */

#define FV_BLK 64

typedef struct {
  int n;
  int64_t len[OR_MAXR];
  int64_t s1[OR_MAXR];       /* stride in the first tensor carrying the group */
  int64_t s2[OR_MAXR];       /* stride in the second tensor carrying the group */
} fv_group;

/* I = C∩A (C order), J = C∩B (C order), P = A∩B (A order), after the same label checks as
 * classify(). For I: s1 = stride in A, s2 = stride in C. J: s1 = B, s2 = C. P: s1 = A, s2 = B. */
static int fv_classify(int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                       int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                       int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                       fv_group* I, fv_group* J, fv_group* P) {
  or_group F, Q;
  int err = classify(rA, lA, sA, labA, rB, lB, sB, labB, rC, lC, sC, labC, &F, &Q);
  if (err) return err;
  I->n = J->n = P->n = 0;
  for (int i = 0; i < rC; ++i) {
    int ia = find(labA, rA, labC[i]);
    if (ia >= 0) {
      I->len[I->n] = lC[i]; I->s1[I->n] = sA[ia]; I->s2[I->n] = sC[i]; I->n++;
    } else {
      int ib = find(labB, rB, labC[i]);
      J->len[J->n] = lC[i]; J->s1[J->n] = sB[ib]; J->s2[J->n] = sC[i]; J->n++;
    }
  }
  for (int i = 0; i < Q.n; ++i) {
    P->len[i] = Q.len[i]; P->s1[i] = Q.sa[i]; P->s2[i] = Q.sb[i];
  }
  P->n = Q.n;
  return 0;
}

static int64_t fv_extent(const fv_group* g) {
  int64_t n = 1;
  for (int i = 0; i < g->n; ++i) n *= g->len[i];
  return n;
}

/* off1[q], off2[q]: location part of group g at linear index q (colexicographic, first fastest),
 * in the first and second tensor carrying g. */
static void fv_offsets(const fv_group* g, int64_t n, int64_t* off1, int64_t* off2) {
  for (int64_t q = 0; q < n; ++q) {
    int64_t r = q, o1 = 0, o2 = 0;
    for (int i = 0; i < g->n; ++i) {
      int64_t x = r % g->len[i];
      r /= g->len[i];
      o1 += x * g->s1[i]; o2 += x * g->s2[i];
    }
    off1[q] = o1; off2[q] = o2;
  }
}

static double fv_load(int dtype, const void* T, int64_t loc) {
  return dtype == 0 ? ((const double*)T)[loc] : (double)((const float*)T)[loc];
}

/* y[r] = sum_{q=0}^{nQ-1} T[offR[r] + offQ[q]] * z[q], for r in [0, nR). */
static void fv_matvec(int dtype, const void* T, const int64_t* offR, int64_t nR,
                      const int64_t* offQ, int64_t nQ, const double* z, double* y) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r0 = 0; r0 < nR; r0 += FV_BLK) {
    int64_t r1 = r0 + FV_BLK < nR ? r0 + FV_BLK : nR;
    double acc[FV_BLK];
    for (int64_t r = r0; r < r1; ++r) acc[r - r0] = 0.0;
    for (int64_t q = 0; q < nQ; ++q) {
      double zq = z[q];
      int64_t oq = offQ[q];
      for (int64_t r = r0; r < r1; ++r) acc[r - r0] += fv_load(dtype, T, offR[r] + oq) * zq;
    }
    for (int64_t r = r0; r < r1; ++r) y[r] = acc[r - r0];
  }
}

/* Group extents (nI, nJ, nP) of a contraction, for sizing the Freivalds vectors. */
int oracle_freivalds_dims(int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                          int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                          int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                          int64_t* dims) {
  fv_group I, J, P;
  int err = fv_classify(rA, lA, sA, labA, rB, lB, sB, labB, rC, lC, sC, labC, &I, &J, &P);
  if (err) return err;
  dims[0] = fv_extent(&I); dims[1] = fv_extent(&J); dims[2] = fv_extent(&P);
  return 0;
}

/* C_new and C_old carry the same labels and lengths (strides may differ: sCold). */
int oracle_freivalds(int dtype,
                     const void* A, int rA, const int64_t* lA, const int64_t* sA, const char* labA,
                     const void* B, int rB, const int64_t* lB, const int64_t* sB, const char* labB,
                     const void* Cnew, int rC, const int64_t* lC, const int64_t* sC, const char* labC,
                     const void* Cold, const int64_t* sCold,
                     const double* x, double* u, double* v, double* wnew, double* wold,
                     int nthreads) {
  fv_group I, J, P;
  int err = fv_classify(rA, lA, sA, labA, rB, lB, sB, labB, rC, lC, sC, labC, &I, &J, &P);
  if (err) return err;
  int64_t nI = fv_extent(&I), nJ = fv_extent(&J), nP = fv_extent(&P);
  int64_t* oIA = malloc(sizeof(int64_t) * (nI ? nI : 1));
  int64_t* oIC = malloc(sizeof(int64_t) * (nI ? nI : 1));
  int64_t* oJB = malloc(sizeof(int64_t) * (nJ ? nJ : 1));
  int64_t* oJC = malloc(sizeof(int64_t) * (nJ ? nJ : 1));
  int64_t* oPA = malloc(sizeof(int64_t) * (nP ? nP : 1));
  int64_t* oPB = malloc(sizeof(int64_t) * (nP ? nP : 1));
  if (!oIA || !oIC || !oJB || !oJC || !oPA || !oPB) {
    free(oIA); free(oIC); free(oJB); free(oJC); free(oPA); free(oPB);
    return 4;
  }
  fv_offsets(&I, nI, oIA, oIC);
  fv_offsets(&J, nJ, oJB, oJC);
  fv_offsets(&P, nP, oPA, oPB);
  set_threads(nthreads);
  fv_matvec(dtype, B, oPB, nP, oJB, nJ, x, u);          /* u = B x      */
  fv_matvec(dtype, A, oIA, nI, oPA, nP, u, v);          /* v = A u      */
  fv_matvec(dtype, Cnew, oIC, nI, oJC, nJ, x, wnew);    /* wnew = Cnew x */
  if (Cold) {                                           /* wold = Cold x */
    fv_group Jo = J, Io = I;
    for (int i = 0, a = 0, b = 0; i < rC; ++i) {        /* C_old's own strides, same labels */
      if (find(labA, rA, labC[i]) >= 0) Io.s2[a++] = sCold[i];
      else Jo.s2[b++] = sCold[i];
    }
    fv_offsets(&Io, nI, oIA, oIC);
    fv_offsets(&Jo, nJ, oJB, oJC);
    fv_matvec(dtype, Cold, oIC, nI, oJC, nJ, x, wold);
  }
  free(oIA); free(oIC); free(oJB); free(oJC); free(oPA); free(oPB);
  return 0;
}
