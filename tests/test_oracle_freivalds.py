"""Pins for the Freivalds full-tensor check (pin p8; oracle_freivalds in
oracle/contract.c) against what the mathematics fixes -- never against the oracle itself.
CPU only.

  * the four matrix-vector products equal numpy matmul (BLAS) on the matrix forms that
    numpy.transpose + reshape(order='F') build from the tensors (§6.1: the colexicographic
    linearisation of each label group), bitwise with integer inputs;
  * a correct C passes exactly (integer inputs) and every single-element corruption of C fails it
    (detection, Freivalds 1977);
  * plausible mistakes fail: a transposed operand, a dropped beta term, a wrong alpha, C_old read
    when beta = 0 (C_old = NaN must not matter);
  * the float residual test sits far below 1e-12 for a correct result and far above it for a
    corrupted one.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads as W


def _groups(case):
    lab_i = [x for x in case.lab_c if x in case.lab_a]
    lab_j = [x for x in case.lab_c if x in case.lab_b]
    lab_p = [x for x in case.lab_a if x in case.lab_b]
    return lab_i, lab_j, lab_p


def _matrix(T, labels, rows, cols, lens):
    """Matrix form of tensor T (labels) with rows = colex over `rows`, cols = colex over `cols`."""
    arr = np.asarray(T, dtype=np.float64)
    axes = [labels.index(x) for x in rows + cols]
    nr = math.prod(lens[x] for x in rows)
    nc = math.prod(lens[x] for x in cols)
    return arr.transpose(axes).reshape((nr, nc), order="F")


def _cases():
    out = [W.random_tiny_case(s, max_rank=6, max_len=5) for s in range(40)]
    out += [W.cfg1().scaled({x: 4 for x in "abcdef"}), W.cfg5(big=4, small=3),
            W.cfg3(True, v=6, o=3), W.cfg2(True, n=9)]
    return out


@pytest.mark.parametrize("k", range(44))
def test_p8_products_equal_blas_on_matrix_forms(k):
    case = _cases()[k]
    case.c_init = "dist"
    if case.beta == 0.0:
        case.beta = 0.5
    A, B, C = W.make_tensors(case)
    lab_i, lab_j, lab_p = _groups(case)
    nI, nJ, nP = oracle.freivalds_dims(case.spec, A, B, C)
    assert (nI, nJ, nP) == tuple(math.prod(case.lens[x] for x in g) for g in (lab_i, lab_j, lab_p))
    Am = _matrix(A, case.lab_a, lab_i, lab_p, case.lens)
    Bm = _matrix(B, case.lab_b, lab_p, lab_j, case.lens)
    Cm = _matrix(C, case.lab_c, lab_i, lab_j, case.lens)
    Cnew = C * 3.0 - 1.0
    Cnm = _matrix(Cnew, case.lab_c, lab_i, lab_j, case.lens)
    x = np.random.RandomState(k).uniform(-1, 1, nJ)
    r = oracle.freivalds(case.spec, A, B, Cnew, C, x)
    u = Bm @ x
    for got, ref in ((r["u"], u), (r["v"], Am @ r["u"]), (r["wnew"], Cnm @ x),
                     (r["wold"], Cm @ x)):
        assert got.shape == ref.shape
        scale = max(1.0, float(np.abs(ref).max()) if ref.size else 1.0)
        assert np.all(np.abs(got - ref) <= 1e-13 * scale), case.name


@pytest.mark.parametrize("k", range(44))
def test_p8_integer_products_bitwise(k):
    case = _cases()[k]
    case.dist, case.c_init = "int", "dist"
    A, B, C = W.make_tensors(case)
    lab_i, lab_j, lab_p = _groups(case)
    Am = _matrix(A, case.lab_a, lab_i, lab_p, case.lens)
    Bm = _matrix(B, case.lab_b, lab_p, lab_j, case.lens)
    Cm = _matrix(C, case.lab_c, lab_i, lab_j, case.lens)
    x = oracle.freivalds_vectors(Bm.shape[1], 1, seed=k)[0]
    r = oracle.freivalds(case.spec, A, B, C, C, x)
    assert np.array_equal(r["u"], Bm @ x)
    assert np.array_equal(r["v"], Am @ (Bm @ x))
    assert np.array_equal(r["wnew"], Cm @ x)
    assert np.array_equal(r["wold"], Cm @ x)


def _int_case(seed=3, alpha=0.5, beta=-1.0):
    case = W.random_tiny_case(seed, max_rank=5, max_len=4, dist="int")
    case.alpha, case.beta, case.c_init = alpha, beta, "dist"
    return case


@pytest.mark.parametrize("seed", [1, 3, 8, 12])
def test_p8_correct_result_passes_exactly(seed):
    case = _int_case(seed)
    A, B, C = W.make_tensors(case)
    Cn = torch.from_numpy(oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(),
                                       case.alpha, case.beta))
    assert oracle.freivalds_check(case.spec, A, B, Cn, C, case.alpha, case.beta,
                                  exact=True) == 0.0


@pytest.mark.parametrize("seed", [1, 3])
def test_p8_every_single_element_corruption_is_detected(seed):
    case = _int_case(seed)
    A, B, C = W.make_tensors(case)
    good = torch.from_numpy(oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(),
                                         case.alpha, case.beta))
    assert good.numel() > 1
    flat = good.reshape(-1)
    for e in range(flat.numel()):
        bad = flat.clone()
        bad[e] += 1.0
        assert oracle.freivalds_check(case.spec, A, B, bad.reshape(good.shape), C, case.alpha,
                                      case.beta, exact=True) > 0.0, e


def test_p8_plausible_mistakes_fail():
    case = W.Case("fm", "abij", "abef", "efij", {x: 4 for x in "abefij"}, dist="int",
                  alpha=0.5, beta=1.0, c_init="dist", seed=77)
    A, B, C = W.make_tensors(case)
    good = torch.from_numpy(oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), 0.5, 1.0))
    chk = lambda Cn, **kw: oracle.freivalds_check(case.spec, A, B, Cn, C, **kw)  # noqa: E731
    assert chk(good, alpha=0.5, beta=1.0, exact=True) == 0.0
    # a transposed operand (e and f swapped in A)
    At = A.permute(0, 1, 3, 2)
    bad = torch.from_numpy(oracle.brute(case.spec, At.numpy(), B.numpy(), C.numpy(), 0.5, 1.0))
    assert chk(bad, alpha=0.5, beta=1.0, exact=True) > 0.0
    # dropped beta term, wrong alpha, wrong sign of beta
    assert chk(good - C, alpha=0.5, beta=1.0, exact=True) > 0.0
    assert chk(good, alpha=1.0, beta=1.0, exact=True) > 0.0
    assert chk(good, alpha=0.5, beta=-1.0, exact=True) > 0.0
    # the output stored with two labels exchanged (C_abji instead of C_abij)
    assert chk(good.transpose(2, 3).contiguous(), alpha=0.5, beta=1.0, exact=True) > 0.0


def test_p8_beta_zero_does_not_read_C_old():
    case = W.cfg5(big=4, small=2)
    case.dist = "int"
    A, B, C = W.make_tensors(case)           # C = NaN
    Cn = C.clone()
    oracle.contract(case.spec, A, B, Cn, 1.0, 0.0)
    assert oracle.freivalds_check(case.spec, A, B, Cn, C, 1.0, 0.0, exact=True) == 0.0


def test_p8_float_residual_separates_correct_from_corrupt():
    case = W.cfg5(big=6, small=3)
    A, B, C = W.make_tensors(case)
    Cn = C.clone()
    oracle.contract(case.spec, A, B, Cn, 1.0, 0.0)
    ok = oracle.freivalds_check(case.spec, A, B, Cn, None, 1.0, 0.0)
    assert ok < 1e-14
    bad = Cn.clone()
    bad[2, 1, 3, 0, 2, 1] += 1e-3 * float(Cn.abs().max())
    assert oracle.freivalds_check(case.spec, A, B, bad, None, 1.0, 0.0) > 1e-12


def test_p8_strided_and_negative_stride_views():
    """Sub-views (multi-GPU shards) and reversed storage (numpy negative strides)."""
    case = W.cfg5(big=6, small=3)
    case.dist = "int"
    A, B, C = W.make_tensors(case)
    full = C.clone()
    oracle.contract(case.spec, A, B, full, 1.0, 0.0)
    As, Bs, Cs = A[2:5, 1:4], B[:, 0:3], full[2:5, 1:4, 0:3]
    assert oracle.freivalds_check(case.spec, As, Bs, Cs, None, 1.0, 0.0, exact=True) == 0.0
    An = A.numpy()[::-1]
    Cr = full.numpy()[::-1]
    assert oracle.freivalds_check(case.spec, An, B.numpy(), Cr, None, 1.0, 0.0, exact=True) == 0.0
    assert oracle.freivalds_check(case.spec, An, B.numpy(), full.numpy(), None, 1.0, 0.0,
                                  exact=True) > 0.0


def test_p8_cfg5_integer_bounds_are_exact():
    """in integer mode (|a|,|b| <= 4, |x| <= 1024) every partial sum of the check
    stays below 2^53 at cfg5's full size, so the check is exact."""
    case = W.cfg5()
    m, n, k = case.mnk()
    c_max = 16 * k
    assert c_max * 1024 * n < 2 ** 53
    assert 4 * (4 * 1024 * n) * k < 2 ** 53
