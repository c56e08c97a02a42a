"""Pins for the oracle (oracle/contract.c, oracle.brute, oracle/plan.py) against what the paper
and the mathematics fix -- never against the oracle itself. CPU only.

  p1 brute force on tiny inputs (two independent statements of P:278-281)
  p2 reduction to textbook GEMM (numpy matmul / BLAS) when each bundle has one index
  p3 invariants: storage permutation, relabelling, A<->B swap, C label permutation, linearity
  p4 closed forms: all-ones, one-hot identity, rank-1 factorised operands
  p5 exactness with small integers (bitwise)
  p6 paper-printed values of the worked example (tests/golden/e1_worked_example.json)
  p7 the fp64 dot-product error bound against exact rational arithmetic
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
from oracle import plan
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(x, y):
    x, y = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64)
    d = np.linalg.norm((x - y).ravel())
    n = np.linalg.norm(y.ravel())
    return d / n if n > 0 else d


def run_oracle(case, A, B, C):
    Cn = C.clone()
    oracle.contract(case.spec, A, B, Cn, case.alpha, case.beta)
    return Cn


# ---------------------------------------------------------------------------------------------
# p1 brute force
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(150))
def test_p1_brute_force_random_tiny(seed):
    case = W.random_tiny_case(seed)
    A, B, C = W.make_tensors(case)
    ref = oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), case.alpha, case.beta)
    got = run_oracle(case, A, B, C).numpy()
    assert got.shape == ref.shape
    scale = max(1.0, np.abs(ref).max()) if ref.size else 1.0
    assert np.all(np.abs(got - ref) <= 1e-13 * scale), case


@pytest.mark.parametrize("seed", range(60))
def test_p5_integer_inputs_bitwise(seed):
    case = W.random_tiny_case(seed, dist="int")
    A, B, C = W.make_tensors(case)
    ref = oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), case.alpha, case.beta)
    got = run_oracle(case, A, B, C).numpy()
    assert np.array_equal(got, ref)


def test_p1_cfg1_structure_vs_brute():
    """cfg1's index structure (fig:bench entry 23) at lengths 3 against brute force."""
    case = W.cfg1().scaled({x: 3 for x in "abcdef"})
    A, B, C = W.make_tensors(case)
    ref = oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), case.alpha, case.beta)
    got = run_oracle(case, A, B, C).numpy()
    assert rel(got, ref) < 1e-14


# ---------------------------------------------------------------------------------------------
# p2 GEMM reduction ("ab-ac-cb = GEMM")
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("spec", ["mn-mk-kn", "mn-km-nk", "ab-ac-cb", "nm-mk-kn"])
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (-0.5, 0.5), (2.0, 1.0)])
def test_p2_gemm_reduction(spec, alpha, beta):
    lc, la, lb = spec.split("-")
    free_a = [x for x in la if x in lc][0]
    free_b = [x for x in lb if x in lc][0]
    bound = [x for x in la if x in lb][0]
    lens = {free_a: 37, free_b: 29, bound: 53}
    case = W.Case("g", lc, la, lb, lens, alpha=alpha, beta=beta, c_init="dist", seed=11)
    A, B, C = W.make_tensors(case)
    Am = A.numpy() if la.index(free_a) == 0 else A.numpy().T          # (M, K)
    Bm = B.numpy() if lb.index(bound) == 0 else B.numpy().T          # (K, N)
    Cm = C.numpy() if lc.index(free_a) == 0 else C.numpy().T         # (M, N)
    ref = alpha * (Am @ Bm) + beta * Cm
    got = run_oracle(case, A, B, C).numpy()
    gotm = got if lc.index(free_a) == 0 else got.T
    assert rel(gotm, ref) < 1e-14


def test_p2_gemm_integer_bitwise():
    case = W.Case("gi", "mn", "mk", "kn", {"m": 40, "n": 33, "k": 70}, dist="int",
                  alpha=2.0, beta=-1.0, c_init="dist", seed=5)
    A, B, C = W.make_tensors(case)
    ref = 2.0 * (A.numpy() @ B.numpy()) - C.numpy()
    assert np.array_equal(run_oracle(case, A, B, C).numpy(), ref)


# ---------------------------------------------------------------------------------------------
# p3 invariants
# ---------------------------------------------------------------------------------------------

def _permute_storage(t, lab, perm):
    """Physically re-store tensor t (labels lab) in label order lab[perm] (column-major)."""
    new_lab = "".join(lab[p] for p in perm)
    lens = [t.shape[p] for p in perm]
    flat = torch.empty(math.prod(lens), dtype=t.dtype)
    view = W.colmajor_view(flat, lens)
    view.copy_(t.permute(tuple(int(p) for p in perm)))
    return view, new_lab


@pytest.mark.parametrize("seed", range(25))
def test_p3_storage_permutation_and_swap_invariance(seed):
    """Integer inputs make every order of summation exact, so these must be bitwise."""
    case = W.random_tiny_case(seed, dist="int")
    A, B, C = W.make_tensors(case)
    base = run_oracle(case, A, B, C)
    rs = np.random.RandomState(seed)
    # (i) permute A's and B's storage together with their labels
    pa, pb = rs.permutation(A.dim()), rs.permutation(B.dim())
    A2, la2 = _permute_storage(A, case.lab_a, list(pa))
    B2, lb2 = _permute_storage(B, case.lab_b, list(pb))
    C2 = C.clone()
    oracle.contract(f"{case.lab_c}-{la2}-{lb2}", A2, B2, C2, case.alpha, case.beta)
    assert torch.equal(C2, base)
    # (iv) swap A and B with their labels
    C3 = C.clone()
    oracle.contract(f"{case.lab_c}-{case.lab_b}-{case.lab_a}", B, A, C3, case.alpha, case.beta)
    assert torch.equal(C3, base)
    # (ii) permute C's labels: output permuted identically
    pc = list(rs.permutation(C.dim()))
    C4, lc4 = _permute_storage(C, case.lab_c, pc)
    oracle.contract(f"{lc4}-{case.lab_a}-{case.lab_b}", A, B, C4, case.alpha, case.beta)
    assert torch.equal(C4, base.permute(tuple(int(p) for p in pc)))
    # (iii) consistent relabelling
    mp = dict(zip("abcdefghijklmnopqrstuvwxyz", "zyxwvutsrqponmlkjihgfedcba"))
    rl = lambda s: "".join(mp[x] for x in s)  # noqa: E731
    C5 = C.clone()
    oracle.contract(f"{rl(case.lab_c)}-{rl(case.lab_a)}-{rl(case.lab_b)}", A, B, C5,
                    case.alpha, case.beta)
    assert torch.equal(C5, base)


def test_p3_linearity_in_alpha_beta():
    case = W.random_tiny_case(7, dist="int")
    A, B, C = W.make_tensors(case)
    spec = case.spec
    r1, r2, r3 = C.clone(), C.clone(), C.clone()
    oracle.contract(spec, A, B, r1, 1.0, 0.0)
    oracle.contract(spec, A, B, r2, 0.0, 1.0)
    oracle.contract(spec, A, B, r3, 3.0, -2.0)
    assert torch.equal(r3, 3.0 * r1 - 2.0 * r2)
    assert torch.equal(r2, C)


def test_p3_blockwise_subranges_assemble_to_full():
    """Computing free sub-blocks of C on sub-views and assembling equals the full
    result (pins partitioning and the multi-GPU sharding over free labels)."""
    case = W.cfg5(big=6, small=3)
    A, B, C = W.make_tensors(case)
    full = run_oracle(case, A, B, C)
    part = C.clone()
    for a0, a1 in ((0, 3), (3, 6)):
        for b0, b1 in ((0, 2), (2, 6)):
            for c0, c1 in ((0, 5), (5, 6)):
                As = A[a0:a1, b0:b1]
                Bs = B[:, c0:c1]
                Cs = part[a0:a1, b0:b1, c0:c1]
                oracle.contract(case.spec, As, Bs, Cs, case.alpha, case.beta)
    assert torch.equal(part, full)


# ---------------------------------------------------------------------------------------------
# p4 closed forms
# ---------------------------------------------------------------------------------------------

def test_p4_all_ones():
    case = W.Case("ones", "abcd", "aebf", "dfce", {"a": 3, "b": 4, "c": 2, "d": 5, "e": 6, "f": 7},
                  c_init="dist", alpha=0.5, beta=2.0, seed=3)
    _, _, C = W.make_tensors(case)
    A = W.colmajor_view(torch.ones(3 * 6 * 4 * 7, dtype=torch.float64), [3, 6, 4, 7])
    B = W.colmajor_view(torch.ones(5 * 7 * 2 * 6, dtype=torch.float64), [5, 7, 2, 6])
    got = C.clone()
    oracle.contract(case.spec, A, B, got, 0.5, 2.0)
    assert torch.allclose(got, 0.5 * 42 + 2.0 * C, rtol=0, atol=1e-13)


def test_p4_one_hot_identity_gives_permuted_copy():
    """B_{dfce} = delta(d,f)*delta(c,e): C_abcd = A_acbd (a permuted copy of A)."""
    n = 4
    A = W.make_tensors(W.Case("x", "abcd", "aebf", "dfce", {x: n for x in "abcdef"}, seed=9))[0]
    B = torch.zeros(n, n, n, n, dtype=torch.float64)
    for d, c in itertools.product(range(n), range(n)):
        B[d, d, c, c] = 1.0
    C = torch.full((n,) * 4, float("nan"), dtype=torch.float64)
    oracle.contract("abcd-aebf-dfce", A, B, C, 1.0, 0.0)
    # C_abcd = sum_{e,f} A_aebf B_dfce = A_a c b d
    assert torch.equal(C, A.permute(0, 2, 1, 3))


def test_p4_rank_one_factorised():
    """A_{aebf} = u_{ab} x_{ef}, B_{dfce} = v_{ef} y_{cd} => C = (x.v) u (x) y."""
    rs = np.random.RandomState(0)
    u, y = rs.randn(3, 4), rs.randn(2, 5)
    x, v = rs.randn(6, 7), rs.randn(6, 7)
    A = torch.from_numpy(np.einsum("ab,ef->aebf", u, x).copy())
    B = torch.from_numpy(np.einsum("ef,cd->dfce", v, y).copy())
    C = torch.zeros(3, 4, 2, 5, dtype=torch.float64)
    oracle.contract("abcd-aebf-dfce", A, B, C, 1.0, 0.0)
    ref = float((x * v).sum()) * np.einsum("ab,cd->abcd", u, y)
    assert rel(C.numpy(), ref) < 1e-14


# ---------------------------------------------------------------------------------------------
# semantics: alpha/beta reads (R1), zero-length (R8), scalars, errors (R6)
# ---------------------------------------------------------------------------------------------

def test_beta_zero_does_not_read_C_and_alpha_zero_does_not_read_AB():
    case = W.cfg1().scaled({x: 3 for x in "abcdef"})
    A, B, C = W.make_tensors(case)
    assert torch.isnan(C).all()
    out = run_oracle(case, A, B, C)
    assert torch.isfinite(out).all()
    An = torch.full_like(A, float("nan"))
    Cv = torch.ones_like(C)
    Bn = torch.full_like(B, float("nan"))
    oracle.contract(case.spec, An, Bn, Cv, 0.0, 3.0)
    assert torch.equal(Cv, torch.full_like(C, 3.0))


def test_zero_length_bundles():
    A = torch.zeros(3, 0, dtype=torch.float64)
    B = torch.zeros(0, 4, dtype=torch.float64)
    C = torch.ones(3, 4, dtype=torch.float64)
    oracle.contract("ab-ak-kb", A, B, C, 1.0, 0.5)          # n_P = 0 -> C = beta C
    assert torch.equal(C, torch.full((3, 4), 0.5, dtype=torch.float64))
    C0 = torch.zeros(0, 4, dtype=torch.float64)
    oracle.contract("ab-ak-kb", torch.zeros(0, 5, dtype=torch.float64),
                    torch.zeros(5, 4, dtype=torch.float64), C0, 1.0, 0.5)


def test_scalar_spec_example():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["contract_naive"][0]
    C = np.array(g["c0"])
    oracle.contract("--", np.array(g["a"]), np.array(g["b"]), C, g["alpha"], g["beta"])
    assert float(C) == g["value"]
    mk = json.load(open(os.path.join(GOLD, "spec_examples.json")))["microkernel"][0]
    C = np.zeros(())
    oracle.contract("-k-k", np.array(mk["a"], dtype=np.float64), np.array(mk["b"], dtype=np.float64), C)
    assert float(C) == mk["value"]


@pytest.mark.parametrize("spec,shapes", [
    ("ad-ab-bc", ([2, 3], [3, 4], [2, 5])),     # d only in C, c only in B
    ("abc-abk-kbc", ([2, 3, 4], [2, 3, 5], [5, 3, 4])),  # b in all three
    ("aa-ak-ka", ([2, 2], [2, 3], [3, 2])),     # repeated label
])
def test_label_errors(spec, shapes):
    A, B, C = (np.zeros(s) for s in shapes)
    with pytest.raises(ValueError):
        oracle.contract(spec, A, B, C)


def test_shape_error():
    with pytest.raises(ValueError):
        oracle.contract("ab-ak-kb", np.zeros((2, 3)), np.zeros((4, 5)), np.zeros((2, 5)))


def test_negative_strides_numpy():
    rs = np.random.RandomState(1)
    a, b = rs.randn(5, 6), rs.randn(6, 7)
    c = np.zeros((5, 7))
    oracle.contract("mn-mk-kn", a[::-1], b[:, ::-1], c)
    assert rel(c, a[::-1] @ b[:, ::-1]) < 1e-14


def test_contract_at_matches_full():
    case = W.cfg4(3).scaled({x: max(2, n // 32) for x, n in W.cfg4(3).lens.items()})
    case.beta, case.c_init = 0.5, "dist"
    A, B, C = W.make_tensors(case)
    full = run_oracle(case, A, B, C)
    rs = np.random.RandomState(0)
    idx = np.stack([rs.randint(0, n, 40) for n in C.shape], axis=1)
    got = oracle.contract_at(case.spec, A, B, C, case.alpha, case.beta, idx)
    ref = np.array([float(full[tuple(i)]) for i in idx])
    assert np.array_equal(got, ref)


def test_fp32_accumulates_in_fp64_rounds_once():
    case = W.random_tiny_case(3, dtype=torch.float32)
    case.lens = {x: 6 for x in case.lens}
    A, B, C = W.make_tensors(case)
    got = C.clone()
    oracle.contract(case.spec, A, B, got, case.alpha, case.beta)
    ref = oracle.brute(case.spec, A.double().numpy(), B.double().numpy(), C.double().numpy(),
                       case.alpha, case.beta)
    assert np.all(np.abs(got.numpy().astype(np.float64) - ref) <= 1e-6 * max(1, np.abs(ref).max()))


# ---------------------------------------------------------------------------------------------
# p7 error bound vs exact arithmetic
# ---------------------------------------------------------------------------------------------

def test_p7_dot_product_error_bound_exact_rationals():
    """|C_oracle - C_exact| <= gamma_K * sum|a||b| with gamma_K = K u / (1 - K u), u = 2^-53;
    C_exact computed in exact rational arithmetic for sampled elements."""
    case = W.Case("p7", "mn", "mk", "kn", {"m": 6, "n": 5, "k": 2048}, seed=77)
    A, B, C = W.make_tensors(case)
    out = run_oracle(case, A, B, C)
    u = 2.0 ** -53
    K = 2048
    gamma = K * u / (1 - K * u)
    a, b = A.numpy(), B.numpy()
    for i, j in [(0, 0), (5, 4), (3, 2)]:
        exact = sum(Fraction(float(a[i, p])) * Fraction(float(b[p, j])) for p in range(K))
        bound = gamma * float(np.sum(np.abs(a[i]) * np.abs(b[:, j])))
        assert abs(Fraction(float(out[i, j])) - exact) <= Fraction(bound)


# ---------------------------------------------------------------------------------------------
# p6 the paper's worked example (planner steps a1-a4)
# ---------------------------------------------------------------------------------------------

def _e1():
    g = json.load(open(os.path.join(GOLD, "e1_worked_example.json")))
    shp = g["shapes"]
    lens = {}
    for t, lab in (("A", "cfbd"), ("B", "fea"), ("C", "abcde")):
        for x, n in zip(lab, shp[t]):
            assert lens.setdefault(x, n) == n          # P:325-326 consistent with eq:ex-contraction
    return g, lens


def test_p6_e1_bundles_and_strides():
    g, lens = _e1()
    sa, sb, sc = (W.colmajor_strides([lens[x] for x in lab]) for lab in ("cfbd", "fea", "abcde"))
    assert sc == g["strides_C"]["value"]
    I, J, P = plan.classify("cfbd", [lens[x] for x in "cfbd"], sa, "fea", [lens[x] for x in "fea"],
                            sb, "abcde", [lens[x] for x in "abcde"], sc)
    assert set("".join(d["labels"] for d in I)) == set(g["bundles"]["I"])
    assert set("".join(d["labels"] for d in J)) == set(g["bundles"]["J"])
    assert set("".join(d["labels"] for d in P)) == set(g["bundles"]["P"])
    nI, nJ, nP = (math.prod(d["len"] for d in X) for X in (I, J, P))
    assert [nI, nJ, nP] == g["n_I_n_J_n_P"]["value"]


def _e1_scatter(lens, order):
    sc = dict(zip("abcde", W.colmajor_strides([lens[x] for x in "abcde"])))
    return plan.scatter([(lens[x], sc[x]) for x in order])


def test_p6_e1_scatter_vectors():
    g, lens = _e1()
    cscat = _e1_scatter(lens, g["cscat_C_prefix"]["J_order"])
    assert cscat[:12] == g["cscat_C_prefix"]["value"]
    rscat = _e1_scatter(lens, g["rscat_C_local_stride"]["I_order"])
    s = g["rscat_C_local_stride"]["value"]
    assert rscat[1] - rscat[0] == s and rscat[2] - rscat[1] == s
    # P:541-546 formulas, term by term
    na, nb, nc, nd = lens["a"], lens["b"], lens["c"], lens["d"]
    for Ib in range(18):
        c, d, b = Ib % nc, (Ib // nc) % nd, (Ib // (nc * nd)) % nb
        assert rscat[Ib] == c * na * nb + d * na * nb * nc + b * na
    for Jb in range(24):
        a, e = Jb % na, (Jb // na) % lens["e"]
        assert cscat[Jb] == a + e * na * nb * nc * nd


def test_p6_e1_scatter_identity_all_432_elements():
    """loc(C_IJ) = rscat_I(C) + cscat_J(C) for every element, against numpy's own
    column-major offsets of C_abcde."""
    g, lens = _e1()
    rscat = _e1_scatter(lens, "cdb")
    cscat = _e1_scatter(lens, "ae")
    shape = [lens[x] for x in "abcde"]
    seen = set()
    for Ib in range(18):
        c, d, b = Ib % lens["c"], (Ib // lens["c"]) % lens["d"], Ib // (lens["c"] * lens["d"])
        for Jb in range(24):
            a, e = Jb % lens["a"], Jb // lens["a"]
            off = int(np.ravel_multi_index((a, b, c, d, e), shape, order="F"))
            assert rscat[Ib] + cscat[Jb] == off
            seen.add(off)
    assert len(seen) == 432


def test_p6_e1_53_percent_constant_stride_microtiles():
    g, lens = _e1()
    mr = g["constant_stride_microtile_percent"]["mR"]
    nr = g["constant_stride_microtile_percent"]["nR"]
    rbs = plan.block_scatter(_e1_scatter(lens, "cdb"), mr)
    cbs = plan.block_scatter(_e1_scatter(lens, "ae"), nr)
    both = sum(1 for r in rbs for c in cbs if r > 0 and c > 0)
    assert round(100 * both / (len(rbs) * len(cbs))) == g["constant_stride_microtile_percent"]["value"]


def test_spec_examples_planner():
    s = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in s["new_column_major"]:
        assert W.colmajor_strides(ex["lens"]) == ex["strides"]
    for ex in s["element_offset"]:
        assert sum(i * t for i, t in zip(ex["idx"], ex["strides"])) == ex["offset"]
    for ex in s["compute_scatter"]:
        v = plan.scatter([tuple(d) for d in ex["dims"]])
        assert v[:len(ex.get("prefix", ex.get("value")))] == ex.get("prefix", ex.get("value"))
    for ex in s["compute_block_scatter"]:
        sc = ex["scat"] if "scat" in ex else plan.scatter([tuple(d) for d in ex["scat_dims"]])
        assert plan.block_scatter(sc, ex["b"]) == ex["value"]
    for ex in s["derive_plan"]:
        la, lb, lc = ex["A"], ex["B"], ex["C"]
        n = lambda lab: [2] * len(lab)  # noqa: E731
        st = lambda lab: W.colmajor_strides(n(lab))  # noqa: E731
        if "error" in ex:
            with pytest.raises(plan.LabelError):
                plan.classify(la, n(la), st(la), lb, n(lb), st(lb), lc, n(lc), st(lc))
            continue
        I, J, P = plan.classify(la, n(la), st(la), lb, n(lb), st(lb), lc, n(lc), st(lc))
        for X, key in ((I, "I"), (J, "J"), (P, "P")):
            assert set("".join(d["labels"] for d in X)) == set(ex[key])
    # fold_and_reorder on E1
    g, lens = _e1()
    tabs = plan.plan_tables("cfbd", [lens[x] for x in "cfbd"],
                            W.colmajor_strides([lens[x] for x in "cfbd"]),
                            "fea", [lens[x] for x in "fea"], W.colmajor_strides([lens[x] for x in "fea"]),
                            "abcde", [lens[x] for x in "abcde"],
                            W.colmajor_strides([lens[x] for x in "abcde"]))
    ex = s["fold_and_reorder"][0]
    assert tabs["swapped"] == ex["swapped"]
    # after the swap the roles exchange: new J = old I sorted by C stride -> (b, c, d) = "bcd"
    # (c, d are contiguous in C but not in A: s_d(A) = 24 != s_c(A)*n_c = 2, so no fold)
    assert "".join(d["labels"] for d in tabs["J"]) == "bcd"
    assert "".join(d["labels"] for d in tabs["I"]) == ex["J_sorted"]
    # partition example: element (0,0) of rows [0,8), cols [8,16) of C with I=cdb, J=ae
    p = s["partition"][0]
    assert _e1_scatter(lens, "cdb")[0] + _e1_scatter(lens, "ae")[8] == p["elem00_offset"]
    assert oracle.flops("abcde-cfbd-fea", lens) == s["contract_naive"][1]["flops"]
    assert (s["contract_naive"][1]["flops"] / 2) ** (1 / 3) == pytest.approx(
        s["effective_lengths"][0]["square"])


# ---------------------------------------------------------------------------------------------
# plan invariants and the plan's tables reproduce the contraction
# ---------------------------------------------------------------------------------------------

def _tables(case):
    lens = case.lens
    args = []
    for lab in (case.lab_a, case.lab_b, case.lab_c):
        ln = [lens[x] for x in lab]
        args += [lab, ln, W.colmajor_strides(ln)]
    return plan.plan_tables(*args)


@pytest.mark.parametrize("seed", range(40))
def test_plan_tables_reproduce_contraction(seed):
    """Gathering A, B, C through the six scatter vectors and multiplying the gathered matrices
    gives the brute-force contraction: pins a1-a3 together."""
    case = W.random_tiny_case(seed, dist="int")
    A, B, C = W.make_tensors(case)
    t = _tables(case)
    # the flat storage of each column-major tensor
    flat = lambda T: torch.as_strided(T, (T.numel(),), (1,)).numpy()  # noqa: E731
    a, b, c = flat(A), flat(B), flat(C)
    if t["swapped"]:
        a, b = b, a
    rA, cA, rB, cB, rC, cC = (np.array(t[k], dtype=np.int64) for k in
                              ("rscat_A", "cscat_A", "rscat_B", "cscat_B", "rscat_C", "cscat_C"))
    Am = a[rA[:, None] + cA[None, :]]
    Bm = b[rB[:, None] + cB[None, :]]
    Cm = c[rC[:, None] + cC[None, :]]
    new = case.alpha * (Am @ Bm) + (case.beta * Cm if case.beta != 0 else 0.0)
    out = c.copy()
    out[rC[:, None] + cC[None, :]] = new
    ref = oracle.brute(case.spec, A.numpy(), B.numpy(), C.numpy(), case.alpha, case.beta)
    assert np.array_equal(out, np.asarray(ref).reshape(-1, order="F"))


@pytest.mark.parametrize("seed", range(40))
def test_plan_heuristic_invariants(seed):
    case = W.random_tiny_case(seed)
    t = _tables(case)
    I, J, P = t["I"], t["J"], t["P"]
    # products preserved
    m, n, k = case.mnk()
    if t["swapped"]:
        m, n = n, m
    assert math.prod(d["len"] for d in I) == m
    assert math.prod(d["len"] for d in J) == n
    assert math.prod(d["len"] for d in P) == k
    # no length-1 dims remain (step 1)
    assert all(d["len"] != 1 for d in I + J + P)
    # unit C-stride, if any I/J dim has one, is on I's first dim
    if any(abs(d["stride"]["C"]) == 1 for d in I + J) and any(d["stride"]["C"] == 1 for d in I + J):
        assert I and I[0]["stride"]["C"] == 1
    # idempotence: normalising the normalised plan changes nothing
    I2, J2, P2, sw2 = plan.normalize(I, J, P)
    assert not sw2 and I2 == I and J2 == J and P2 == P


def test_plan_no_simultaneous_stride1_counterexample():
    """C_ijk := A_jli B_lk: no dim has stride 1 in both A and C."""
    lens = {"i": 3, "j": 4, "k": 5, "l": 6}
    args = []
    for lab in ("jli", "lk", "ijk"):
        ln = [lens[x] for x in lab]
        args += [lab, ln, W.colmajor_strides(ln)]
    I, J, P = plan.classify(*args)
    assert not any(d["stride"]["A"] == 1 and d["stride"]["C"] == 1 for d in I)
