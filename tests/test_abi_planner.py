"""Host-side checks of the C ABI library (no GPU needed): it loads, exports every symbol that
include/tc.h declares, and its planner (steps a1-a4) agrees exactly with the
independent oracle/plan.py on the worked example, the BASELINE configs and random cases."""
import os
import re

import numpy as np
import pytest
import torch

import paper_1607_00291_b200 as tc
import workloads as W
from oracle import plan as oplan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "tc.h")).read()
    names = sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tc_\w+)\s*\(", hdr, re.M)))
    assert names and set(names) == set(tc.EXPORTS)
    for n in names:
        assert hasattr(tc._lib, n), n
    assert tc.version() == 100


def _shapes(case):
    out = []
    for lab in (case.lab_a, case.lab_b, case.lab_c):
        ln = [case.lens[x] for x in lab]
        out.append((lab, ln, W.colmajor_strides(ln)))
    return out


def _compare(case):
    (la, sa, ta), (lb, sb, tb), (lc, sc, tcs) = _shapes(case)
    p = tc.Plan(case.spec, case.dtype, (sa, sb, sc), (ta, tb, tcs))
    ref = oplan.plan_tables(la, sa, ta, lb, sb, tb, lc, sc, tcs)
    info = p.info()
    assert info["swapped"] == ref["swapped"]
    for which, key, k0, k1 in ((0, "I", "A", "C"), (1, "J", "B", "C"), (2, "P", "A", "B")):
        got = p.dims(which)
        exp = [(d["labels"], d["len"], d["stride"][k0], d["stride"][k1]) for d in ref[key]]
        assert got == exp, (key, got, exp)
    for i, name in enumerate(tc.SCATTER_NAMES):
        assert p.scatter(i) == ref[name], name
        for b in (2, 4, 8, 16):
            assert p.block_scatter(i, b) == oplan.block_scatter(ref[name], b), (name, b)
    m, n, k = (int(np.prod([d["len"] for d in ref[x]])) for x in ("I", "J", "P"))
    assert (info["m"], info["n"], info["k"]) == (m, n, k)
    return p, ref


def test_planner_worked_example_matches_oracle_and_paper():
    case = W.Case("e1", "abcde", "cfbd", "fea", {"a": 6, "b": 3, "c": 2, "d": 3, "e": 4, "f": 4})
    p, ref = _compare(case)
    assert p.info()["swapped"]
    # c, d are sequentially contiguous in C (fig:bsm caption) but not in A
    # (s_d(A) = 24 != s_c(A) n_c = 2), so step 2 does not fold them: J = (b, c, d)
    assert [d[0] for d in p.dims(1)] == ["b", "c", "d"]


@pytest.mark.parametrize("maker", [W.cfg1, lambda: W.cfg2(False), lambda: W.cfg2(True),
                                   lambda: W.cfg3(False, 8, 4), lambda: W.cfg3(True, 8, 4),
                                   lambda: W.cfg5(6, 3)])
def test_planner_baseline_structures(maker):
    case = maker()
    if case.lens.get("m", 0) > 64:
        case = case.scaled({x: 64 for x in case.lens})
    _compare(case)


def test_planner_folds_cfg3_to_plain_gemm():
    p, _ = _compare(W.cfg3(False, 8, 4))
    assert p.info()["ndims"] == [1, 1, 1]                     # ab, ij, ef each fold (§8 table)


@pytest.mark.parametrize("i", range(20))
def test_planner_cfg4_structures(i):
    case = W.cfg4(i)
    small = case.scaled({x: max(1, min(n, 7)) for x, n in case.lens.items()})
    _compare(small)
    (la, sa, ta), (lb, sb, tb), (lc, sc, tcs) = _shapes(case)
    p = tc.Plan(case.spec, case.dtype, (sa, sb, sc), (ta, tb, tcs))
    ref = oplan.plan_tables(la, sa, ta, lb, sb, tb, lc, sc, tcs)
    for i2, name in enumerate(tc.SCATTER_NAMES):       # full-size tables, exact
        assert p.scatter(i2) == ref[name]


@pytest.mark.parametrize("seed", range(120))
def test_planner_random_tiny(seed):
    _compare(W.random_tiny_case(seed))


@pytest.mark.parametrize("seed", range(40))
def test_planner_random_strided_views(seed):
    """Non-column-major layouts: random sub-views with gaps and negative-free strides."""
    case = W.random_tiny_case(seed, max_len=4)
    rs = np.random.RandomState(seed)
    shapes = []
    for lab in (case.lab_a, case.lab_b, case.lab_c):
        ln = [case.lens[x] for x in lab]
        order = rs.permutation(len(ln))
        st, s = [0] * len(ln), 1
        for d in order:
            st[d] = s
            s *= ln[d] + int(rs.randint(0, 2))
        shapes.append((lab, ln, st))
    (la, sa, ta), (lb, sb, tb), (lc, sc, tcs) = shapes
    p = tc.Plan(case.spec, torch.float64, (sa, sb, sc), (ta, tb, tcs))
    ref = oplan.plan_tables(la, sa, ta, lb, sb, tb, lc, sc, tcs)
    assert p.info()["swapped"] == ref["swapped"]
    for i, name in enumerate(tc.SCATTER_NAMES):
        assert p.scatter(i) == ref[name]


@pytest.mark.parametrize("spec,shapes,code", [
    ("ad-ab-bc", ([2, 3], [3, 4], [2, 5]), 2),
    ("abc-abk-kbc", ([2, 3, 4], [2, 3, 5], [5, 3, 4]), 2),
    ("aa-ak-ka", ([2, 2], [2, 3], [3, 2]), 2),
    ("ab-ak-kb", ([2, 3], [4, 5], [2, 5]), 3),
])
def test_planner_errors(spec, shapes, code):
    st = [W.colmajor_strides(s) for s in shapes]
    with pytest.raises(tc.TCError) as e:
        tc.Plan(spec, torch.float64, shapes, st)
    assert e.value.code == code


def test_planner_rejects_non_injective_output():
    with pytest.raises(tc.TCError) as e:
        tc.Plan("ab-ak-kb", torch.float64, ([3, 4], [4, 5], [3, 5]), ([1, 3], [1, 4], [1, 1]))
    assert e.value.code == 4
    with pytest.raises(tc.TCError) as e:
        tc.Plan("ab-ak-kb", torch.float64, ([3, 4], [4, 5], [3, 5]), ([1, 3], [1, 4], [0, 3]))
    assert e.value.code == 4


def test_planner_rank_limit():
    labs = "abcdefghijklmnopq"  # 17 labels
    with pytest.raises(tc.TCError) as e:
        tc.Plan(f"{labs}-{labs[:9]}-{labs[9:]}", torch.float64,
                ([1] * 9, [1] * 8, [1] * 17), ([1] * 9, [1] * 8, [1] * 17))
    assert e.value.code in (2, 5)


@pytest.mark.parametrize("idx", range(24))
def test_planner_fig_bench_structures(idx):
    """The paper's 24 fig:bench index strings at small synthetic sizes."""
    _compare(W.fig_bench(idx, elems=2 ** 10))


@pytest.mark.parametrize("i", range(7))
def test_planner_rankk_structures(i):
    _compare(W.rankk(i, mn=60))


@pytest.mark.parametrize("seed", range(60))
def test_traversal_tables_reproduce_contraction(seed):
    """The kernel's traversal-order tables (reading R16) are a relinearisation of the same
    contraction: gathering through them and multiplying gives the brute-force result."""
    _check_traversal(W.random_tiny_case(seed, max_len=5, dist="int"))


def _check_traversal(case):
    import oracle
    A, B, C = W.make_tensors(case)
    (la, sa, ta), (lb, sb, tb), (lc, sc, tcs) = _shapes(case)
    p = tc.Plan(case.spec, case.dtype, (sa, sb, sc), (ta, tb, tcs))
    flat = lambda T: torch.as_strided(T, (T.numel(),), (1,)).numpy()  # noqa: E731
    a, b, c = flat(A), flat(B), flat(C)
    if p.info()["swapped"]:
        a, b = b, a
    rA, cA, rB, cB, rC, cC = (np.array(p.traversal_scatter(i), dtype=np.int64) for i in range(6))
    out = c.copy()
    if len(cA):
        new = case.alpha * (a[rA[:, None] + cA[None, :]] @ b[rB[:, None] + cB[None, :]])
    else:
        new = np.zeros((len(rC), len(cC)))
    if case.beta != 0:
        new = new + case.beta * c[rC[:, None] + cC[None, :]]
    out[rC[:, None] + cC[None, :]] = new
    ref = oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), case.alpha, case.beta)
    assert np.array_equal(out, np.asarray(ref).reshape(-1, order="F"))
    # and it is the paper-order table set up to a permutation of rows/columns
    for i in range(6):
        assert sorted(p.traversal_scatter(i)) == sorted(p.scatter(i))
    return p


def test_dimension_subdivision_of_the_long_bundle():
    """f4: fig:bench's abcde-efbad-cf shape class at lengths 4 -- A's unit-stride
    index e and C's a are both in I; the traversal interleaves a 4 x 4 block of them, so the
    first rows step C by 1 and A by its a-stride, and row 4 is A's next element."""
    lens = {x: 4 for x in "abcdef"}
    case = W.Case("sub_I", "abcde", "efbad", "cf", lens, dist="int", alpha=2.0, beta=0.0,
                  c_init="zero", seed=3)
    p = _check_traversal(case)
    rA, rC = p.traversal_scatter(0), p.traversal_scatter(4)
    assert rC[:4] == [0, 1, 2, 3]
    assert rA[:4] == [0, 64, 128, 192] and rA[4] == 1


def test_dimension_subdivision_of_the_bound_bundle():
    """f4 for P: A's unit-stride bound index k and B's d differ (cfg4 case 5's class,
    roc-krdo-dck); the K traversal takes 4 k then 4 d, so A reads runs of 4 and so does B."""
    lens = {"r": 6, "o": 5, "k": 8, "d": 4, "c": 7}
    case = W.Case("sub_P", "roc", "krdo", "dck", lens, dist="int", alpha=1.0, beta=0.5,
                  c_init="dist", seed=4)
    p = _check_traversal(case)
    cA, rB = p.traversal_scatter(1), p.traversal_scatter(2)
    assert cA[:4] == [0, 1, 2, 3] and rB[4:8] == [1, 1 + 4 * 7, 1 + 2 * 4 * 7, 1 + 3 * 4 * 7]


def test_dimension_subdivision_of_the_bound_bundle_two_levels():
    """f4 for P with both unit-stride lengths multiples of 16 (fig:bench ab-cad-dcb's class):
    the K traversal is [k_lo 4, d_lo 4, k_mid 4, d_mid 4, k_hi, d_hi], so every 16 K steps of
    16 read k 0..15 x d 0..15 -- whole 128-byte lines of both operands."""
    lens = {"r": 3, "o": 2, "k": 32, "d": 48, "c": 5}
    case = W.Case("sub_P2", "roc", "krdo", "dck", lens, dist="int", alpha=1.0, beta=0.5,
                  c_init="dist", seed=6)
    p = _check_traversal(case)
    A, B, _ = W.make_tensors(case)
    sk, sd = A.stride(0), A.stride(2)      # A = krdo
    tk, td = B.stride(2), B.stride(0)      # B = dck
    cA, rB = p.traversal_scatter(1), p.traversal_scatter(2)
    for t in range(32 * 48):
        k = t % 4 + 4 * ((t // 16) % 4) + 16 * ((t // 256) % 2)
        d = (t // 4) % 4 + 4 * ((t // 64) % 4) + 16 * (t // 512)
        assert cA[t] == k * sk + d * sd, t
        assert rB[t] == k * tk + d * td, t
