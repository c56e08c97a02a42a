"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on the
same seeded inputs. Tolerance (BASELINE.json north_star): normwise relative error <= 1e-12 for
fp64 and <= 1e-5 for fp32; bitwise in integer-input mode (pin p5: every partial sum is exact).

Small cases run the full oracle; full BASELINE sizes are checked on sampled sub-blocks (a few
index values per free label, always including 0 and n-1) that the oracle computes exactly as
the full contraction would, in the launch configuration bench.py times."""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-12, torch.float32: 1e-5}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_00291_b200  # noqa: F401  (raises if the native library is missing)


def tc():
    import paper_1607_00291_b200 as m
    return m


@pytest.fixture(params=["0", "1", "128", "256", "pair"],
                ids=["ffma", "umma", "umma128", "umma256", "ummapair"])
def both_f32_paths(request, monkeypatch):
    """fp32 cases through the FFMA2 kernel (TC_F32_UMMA=0) and the tcgen05 3xTF32 kernel in the
    form the library picks (N = 256 unless an operand has vector gathers) and in each form
    forced (TC_UMMA_FORM=128|256|pair); the library reads both variables on every call."""
    if request.param == "0":
        monkeypatch.setenv("TC_F32_UMMA", "0")
    else:
        monkeypatch.setenv("TC_F32_UMMA", "1")
        if request.param != "1":
            monkeypatch.setenv("TC_UMMA_FORM", request.param)
    return request.param


@pytest.fixture(params=["1", "0"], ids=["tiny", "tensorcore"])
def both_small_paths(request, monkeypatch):
    """Small cases run through the tiny kernel (tiny.cu) and, with TC_TINY=0, through the
    tensor-core kernel; the library reads TC_TINY on every call."""
    monkeypatch.setenv("TC_TINY", request.param)
    return request.param


def relerr(got, ref):
    got = np.asarray(got, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    n = np.linalg.norm(ref)
    d = np.linalg.norm(got - ref)
    return d / n if n > 0 else d


def run_both(case):
    """Full oracle on CPU and the CUDA path on the same seeded inputs."""
    A, B, C = W.make_tensors(case, "cpu")
    Ad, Bd, Cd = W.make_tensors(case, "cuda", gen_device="cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    return Cd.cpu(), ref


def check(case, bitwise=False):
    got, ref = run_both(case)
    assert torch.isfinite(got).all(), case.name
    if bitwise:
        assert torch.equal(got, ref), case.name
    else:
        e = relerr(got.numpy(), ref.numpy())
        assert e <= TOL[case.dtype], (case.name, e)
    return got, ref


def sampled_check(case, Ad, Bd, Cd_before, Cd_after, per_label=3, seed=0):
    """Check a sampled sub-block of a full-size result: choose `per_label` indices of every free
    label (incl. 0 and n-1), all indices of every bound label, slice A, B, C to them and run the
    oracle on the sub-problem (identical arithmetic to the full definition for those elements)."""
    rs = np.random.RandomState(seed)
    sel = {}
    for x in case.lab_c:
        n = case.lens[x]
        pick = {0, n - 1} | set(rs.randint(0, n, size=per_label).tolist())
        sel[x] = torch.tensor(sorted(pick))

    def sub(T, labels):
        for d, x in enumerate(labels):
            if x in sel:
                T = T.index_select(d, sel[x].to(T.device))
        return T.cpu().contiguous()

    a, b = sub(Ad, case.lab_a), sub(Bd, case.lab_b)
    c0, c1 = sub(Cd_before, case.lab_c), sub(Cd_after, case.lab_c)
    ref = c0.clone()
    oracle.contract(case.spec, a, b, ref, case.alpha, case.beta)
    return relerr(c1.numpy(), ref.numpy()), c1, ref


# ---------------------------------------------------------------------------------------------
# BASELINE configs (small enough for the full oracle, or scaled with ragged tails)
# ---------------------------------------------------------------------------------------------

@pytest.mark.usefixtures("both_small_paths")
def test_cfg1_full_nan_C_beta0():
    got, _ = check(W.cfg1())
    assert torch.isfinite(got).all()


@pytest.mark.usefixtures("both_small_paths")
def test_cfg1_integer_bitwise():
    case = W.cfg1()
    case.dist = "int"
    check(case, bitwise=True)


@pytest.mark.parametrize("transposed", [False, True])
def test_cfg2_ragged(transposed):
    case = W.cfg2(transposed).scaled({"m": 300, "n": 257, "k": 333})
    check(case)


@pytest.mark.parametrize("transposed", [False, True])
def test_cfg2_full_vs_cublas(transposed):
    """cfg2 at 2048^3: the contraction against cuBLAS DGEMM on the same matrices (P:1216-1238:
    same flops, same data) and against the oracle on sampled blocks."""
    case = W.cfg2(transposed)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    Am = Ad if not transposed else Ad.t()     # (m, k)
    Bm = Bd if not transposed else Bd.t()     # (k, n)
    ref = case.alpha * (Am @ Bm) + case.beta * C0
    assert relerr(Cd.cpu().numpy(), ref.cpu().numpy()) < 1e-12
    e, _, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=40)
    assert e < 1e-12


@pytest.mark.parametrize("variant", [False, True])
def test_cfg3_scaled(variant):
    check(W.cfg3(variant, v=24, o=10))


@pytest.mark.parametrize("variant", [False, True])
def test_cfg3_full_sampled(variant):
    case = W.cfg3(variant)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, _, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=4)
    assert e < 1e-12


def _scaled_cfg4(i, dtype=torch.float64, target=120):
    case = W.cfg4(i, dtype)
    lens = {}
    for x, n in case.lens.items():
        lens[x] = max(2, int(round(n ** 0.6))) if n > 64 else max(2, n // 3)
    return case.scaled(lens)


@pytest.mark.parametrize("i", range(20))
def test_cfg4_scaled_f64(i):
    check(_scaled_cfg4(i))


@pytest.mark.parametrize("i", range(20))
def test_cfg4_full_sampled_f64(i):
    case = W.cfg4(i)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=3, seed=i)
    assert torch.isfinite(c1).all()
    assert e < 1e-12


def test_cfg5_scaled_full():
    check(W.cfg5(big=12, small=6))


@pytest.mark.slow
def test_cfg5_full_sampled():
    """cfg5 at full size (8.45e13 flops, 30.6 GB), as bench.py runs it at N=1."""
    case = W.cfg5()
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=2)
    assert torch.isfinite(c1).all()
    assert e < 1e-12


# ---------------------------------------------------------------------------------------------
# loader paths, layouts and edge cases
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("spec", ["mn-mk-kn", "mn-km-nk", "mn-mk-nk", "mn-km-kn",
                                  "nm-mk-kn", "nm-km-nk"])
def test_all_loader_direction_combinations(spec):
    lc, la, lb = spec.split("-")
    case = W.Case("dir_" + spec, lc, la, lb, {"m": 203, "n": 145, "k": 171}, alpha=-0.75,
                  beta=0.25, c_init="dist", seed=21)
    check(case)
    case.dist = "int"
    case.alpha, case.beta = 2.0, -1.0
    check(case, bitwise=True)


@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("seed", range(30))
def test_random_small_contractions(seed):
    case = W.random_tiny_case(seed, max_rank=6, max_len=7)
    check(case)


@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("seed", range(10))
def test_random_small_integer_bitwise(seed):
    check(W.random_tiny_case(seed, max_rank=6, max_len=7, dist="int"), bitwise=True)


@pytest.mark.usefixtures("both_small_paths")
def test_alpha_zero_does_not_read_A_B():
    case = W.cfg3(False, v=8, o=4)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    Ad.fill_(float("nan")); Bd.fill_(float("nan"))
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, 0.0, 0.5)
    assert torch.equal(Cd, 0.5 * C0)


@pytest.mark.usefixtures("both_small_paths")
def test_zero_length_and_empty_bundles():
    dev = "cuda"
    A = torch.randn(5, 0, dtype=torch.float64, device=dev)
    B = torch.randn(0, 7, dtype=torch.float64, device=dev)
    C = torch.ones(5, 7, dtype=torch.float64, device=dev)
    tc().contract("mn-mk-kn", A, B, C, 1.0, 0.5)          # n_P = 0 -> C = beta C
    assert torch.equal(C, torch.full_like(C, 0.5))
    C0 = torch.ones(0, 7, dtype=torch.float64, device=dev)
    tc().contract("mn-mk-kn", torch.randn(0, 3, dtype=torch.float64, device=dev),
                  torch.randn(3, 7, dtype=torch.float64, device=dev), C0, 1.0, 0.0)
    # outer product (d_P = 0) and full reduction to a scalar (d_I = d_J = 0)
    for spec, sa, sb, sc in (("ab-a-b", [37], [29], [37, 29]), ("-abc-abc", [5, 6, 7], [5, 6, 7], [])):
        A = torch.randn(sa, dtype=torch.float64)
        B = torch.randn(sb, dtype=torch.float64)
        C = torch.zeros(sc, dtype=torch.float64)
        ref = C.clone()
        oracle.contract(spec, A, B, ref, 1.5, 0.0)
        Cd = C.cuda()
        tc().contract(spec, A.cuda(), B.cuda(), Cd, 1.5, 0.0)
        assert relerr(Cd.cpu().numpy(), ref.numpy()) < 1e-13, spec


@pytest.mark.usefixtures("both_small_paths")
def test_strided_subviews_and_misaligned_bases():
    """Sub-views with gaps and odd element offsets (16-byte vectors disabled per element)."""
    rs = torch.Generator().manual_seed(3)
    bigA = torch.rand(70, 9, 61, dtype=torch.float64, generator=rs)
    bigB = torch.rand(61, 5, 50, dtype=torch.float64, generator=rs)
    bigC = torch.rand(71, 53, dtype=torch.float64, generator=rs)
    for off in (0, 1):
        A = bigA[off:off + 65, 3, :57]          # (m=65, k=57), strides (549, 1)
        B = bigB[:57, 2, off:off + 47]           # (k, n=47)
        C = bigC[off:off + 65, 1:48]             # (m, n)
        ref = C.clone()
        oracle.contract("mn-mk-kn", A, B, ref, 1.0, -1.0)
        Ad = bigA.cuda()[off:off + 65, 3, :57]
        Bd = bigB.cuda()[:57, 2, off:off + 47]
        bigCd = bigC.cuda()
        Cd = bigCd[off:off + 65, 1:48]
        tc().contract("mn-mk-kn", Ad, Bd, Cd, 1.0, -1.0)
        assert relerr(Cd.cpu().numpy(), ref.numpy()) < 1e-13
        # elements of the big buffer outside the view are untouched
        mask = torch.ones_like(bigC, dtype=torch.bool)
        mask[off:off + 65, 1:48] = False
        assert torch.equal(bigCd.cpu()[mask], bigC[mask])


@pytest.mark.usefixtures("both_small_paths")
def test_storage_permutation_invariance_bitwise():
    """Permuting an operand's storage with its labels gives identical C (pin p3(i), int mode)."""
    base = W.Case("perm", "abij", "abef", "efij", {"a": 20, "b": 11, "e": 9, "f": 13, "i": 6, "j": 7},
                  dist="int", alpha=1.0, beta=0.0, c_init="nan", seed=5)
    got0, _ = run_both(base)
    Ad, Bd, _ = W.make_tensors(base, "cuda", gen_device="cpu")
    for la, perm in (("faeb", (3, 0, 2, 1)), ("ebaf", (2, 1, 0, 3))):
        A2 = W.colmajor_view(torch.empty(Ad.numel(), dtype=Ad.dtype, device="cuda"),
                             [base.lens[x] for x in la])
        A2.copy_(Ad.permute(*perm))
        C = torch.full([base.lens[x] for x in "abij"], float("nan"), dtype=torch.float64, device="cuda")
        tc().contract(f"abij-{la}-efij", A2, Bd, C, 1.0, 0.0)
        assert torch.equal(C.cpu(), got0)


def test_errors_raise_and_enqueue_nothing():
    A = torch.randn(4, 5, dtype=torch.float64, device="cuda")
    B = torch.randn(5, 6, dtype=torch.float64, device="cuda")
    C = torch.zeros(4, 6, dtype=torch.float64, device="cuda")
    with pytest.raises(tc().TCError):
        tc().contract("mn-mk-kq", A, B, C)
    with pytest.raises(tc().TCError):
        tc().contract("mn-mk-kn", A, B, C.as_strided((4, 6), (1, 0)))   # C not injective
    assert torch.equal(C, torch.zeros_like(C))


def test_host_path_end_to_end():
    case = W.cfg3(True, v=20, o=9)
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    Ap, Bp, Cp = A, B, C.clone()
    tc().contract_host(case.spec, Ap, Bp, Cp, case.alpha, case.beta)
    assert relerr(Cp.numpy(), ref.numpy()) < 1e-12


def _host_vs_device(case, C_host_big=None):
    """contract_host on pinned host tensors vs contract on the device, integer inputs (pin p5:
    every partial sum exact, so both must be bitwise equal whatever the chunking)."""
    A, B, C = W.make_tensors(case, "cpu")
    Ap, Bp = A.pin_memory(), B.pin_memory()
    Cp = W.colmajor_view(torch.empty(C.numel(), dtype=C.dtype).pin_memory(), list(C.shape))
    Cp.copy_(C)
    Ad, Bd, Cd = A.cuda(), B.cuda(), C.cuda()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    tc().contract_host(case.spec, Ap, Bp, Cp, case.alpha, case.beta)
    torch.cuda.synchronize()
    assert torch.equal(Cp, Cd.cpu()), case.name
    return A, B, C, Cp


@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_host_path_chunked_cfg5_structure(beta):
    """cfg5's structure at 24/12 (A 191 MB): the host path cuts C into chunks along k (C's and
    B's outermost label) and pipelines copies with kernels; equal to the device path bitwise
    (integer mode) and to the oracle on a sampled sub-block."""
    case = W.cfg5(24, 12)
    case.dist, case.alpha, case.beta, case.c_init = "int", 1.0, beta, "dist"
    A, B, C, Cp = _host_vs_device(case)
    e, c1, _ = sampled_check(case, A, B, C, Cp, per_label=2)
    assert e == 0.0


def test_host_path_chunked_beta_and_scattered_C():
    """cfg3 variant (C stored aibj, beta = 1 so C chunks are uploaded too), 134 MB operands."""
    case = W.cfg3(True, v=64, o=32)
    case.dist, case.alpha, case.beta = "int", 0.5, 1.0
    A, B, C, Cp = _host_vs_device(case)
    e, _, _ = sampled_check(case, A, B, C, Cp, per_label=3)
    assert e == 0.0


def test_host_path_chunked_C_with_holes():
    """C is a sub-view of a larger pinned buffer: chunks along n (C's outer stride) copy spans
    that include the holes, which must come back unchanged."""
    g = torch.Generator().manual_seed(11)
    m, n, k = 4090, 1000, 2048
    A = torch.randint(-4, 5, (k, m), generator=g).double().t()          # (m, k) strides (1, m)
    B = torch.randint(-4, 5, (n, k), generator=g).double().t()          # (k, n) strides (1, k)
    big = torch.randint(-4, 5, (1003, 4096), generator=g).double().pin_memory()
    Cv = big.t()[:m, 1:n + 1]                                            # strides (1, 4096)
    keep = big.clone()
    ref_dev = Cv.cuda()
    tc().contract("mn-mk-kn", A.cuda(), B.cuda(), ref_dev, 2.0, 0.0)
    tc().contract_host("mn-mk-kn", A.pin_memory(), B.pin_memory(), Cv, 2.0, 0.0)
    assert torch.equal(Cv, ref_dev.cpu())
    mask = torch.ones_like(big, dtype=torch.bool)
    mask.t()[:m, 1:n + 1] = False
    assert torch.equal(big[mask], keep[mask])


def test_host_path_release_staging():
    case = W.cfg3(False, v=16, o=8)
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    tc().contract_host(case.spec, A, B, C, case.alpha, case.beta)   # pageable memory
    tc().release_staging()
    assert relerr(C.numpy(), ref.numpy()) < 1e-12


def test_repeat_calls_bitwise_deterministic():
    case = W.cfg4(5)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C1, C2 = Cd.clone(), Cd.clone()
    tc().contract(case.spec, Ad, Bd, C1)
    tc().contract(case.spec, Ad, Bd, C2)
    assert torch.equal(C1, C2)


# ---------------------------------------------------------------------------------------------
# fp32 (cfg4's fp32 half): operands widened to fp64 in the micro-kernel, rounded once (R12)
# ---------------------------------------------------------------------------------------------

@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("i", range(20))
def test_cfg4_scaled_f32(i):
    check(_scaled_cfg4(i, torch.float32))


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("i", range(20))
def test_cfg4_full_sampled_f32(i):
    case = W.cfg4(i, torch.float32)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=3, seed=i)
    assert torch.isfinite(c1).all()
    assert e < TOL[torch.float32]


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("spec", ["mn-mk-kn", "mn-km-nk", "mn-mk-nk", "mn-km-kn"])
@pytest.mark.parametrize("mnk", [(203, 145, 171), (256, 128, 64)])
def test_f32_loader_directions(spec, mnk):
    lc, la, lb = spec.split("-")
    case = W.Case("f32dir_" + spec, lc, la, lb, dict(zip("mnk", mnk)), dtype=torch.float32,
                  alpha=-0.75, beta=0.25, c_init="dist", seed=22)
    check(case)
    case.dist = "int"
    case.alpha, case.beta = 2.0, -1.0
    check(case, bitwise=True)


@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("seed", range(15))
def test_random_small_f32(seed):
    check(W.random_tiny_case(seed, max_rank=6, max_len=7, dtype=torch.float32))


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("spec", ["mn-mk-kn", "mn-km-nk", "mn-mk-nk", "mn-km-kn"])
@pytest.mark.parametrize("mnk", [(260, 196, 100), (132, 388, 36), (516, 132, 260)])
def test_f32_vector_gathers(spec, mnk):
    """Lengths that are multiples of 4 with aligned bases: the plan proves every 16-byte vector
    contiguous, so the tcgen05 kernel's vector gathers run (K vectors into the K-major layout,
    M vectors into the [k][m] staging of A); ragged tiles in M, N and K."""
    lc, la, lb = spec.split("-")
    case = W.Case("f32vec_" + spec, lc, la, lb, dict(zip("mnk", mnk)), dtype=torch.float32,
                  alpha=0.75, beta=-0.5, c_init="dist", seed=41)
    check(case)
    case.dist = "int"
    check(case, bitwise=True)


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("spec", ["mn-mk-kn", "mn-km-nk", "mn-mk-nk", "mn-km-kn"])
@pytest.mark.parametrize("mnk", [(262, 198, 102), (130, 390, 34), (514, 134, 262)])
def test_f32_pair_gathers(spec, mnk):
    """Even lengths that are not multiples of 4: every 8-byte pair of an operand's gather
    direction is contiguous and aligned but its 16-byte vectors are not, so the tcgen05 kernel's
    8-byte pair gathers run (K pairs into the K-major layout, M pairs of A into the [k][m]
    staging); ragged tiles in M, N and K; also at a 4-byte offset (pairs misaligned: element
    gathers)."""
    lc, la, lb = spec.split("-")
    case = W.Case("f32pair_" + spec, lc, la, lb, dict(zip("mnk", mnk)), dtype=torch.float32,
                  alpha=0.75, beta=-0.5, c_init="dist", seed=43)
    info = tc().Plan(case.spec, torch.float32, [case.shape(x) for x in (la, lb, lc)],
                     [W.colmajor_strides(case.shape(x)) for x in (la, lb, lc)]).info()
    assert info["m"] % 2 == 0 and info["k"] % 2 == 0
    check(case)
    case.dist = "int"
    check(case, bitwise=True)
    # the same operands one element off a 16-byte boundary
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    bufA = torch.empty(A.numel() + 1, device="cuda")
    Ad = W.colmajor_view(bufA[1:], list(A.shape))
    Ad.copy_(A.cuda())
    Cd = C.cuda()
    tc().contract(case.spec, Ad, B.cuda(), Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    assert torch.equal(Cd.cpu(), ref)


@pytest.mark.parametrize("shift", ["2", "1", "0"], ids=["shifted", "auto", "elements"])
@pytest.mark.parametrize("lens", [dict(m=300, a=21, b=13, k=7, j=9),
                                  dict(m=130, a=11, b=37, k=5, j=29),
                                  dict(m=517, a=63, b=5, k=33, j=3),
                                  dict(m=64, a=7, b=40, k=3, j=2)])
def test_f32_shifted_n_vectors(lens, shift, monkeypatch):
    """B gathered along N with runs (the unit-stride label a, odd length) that start at every
    4-byte offset: the N = 256 form copies each run as the aligned 16-byte blocks covering it
    and the converter warps pick the values out at the run's shift for each k (umma_f32.cu
    gather mode 12, forced with TC_UMMA_SHIFT=2); TC_UMMA_SHIFT=0 forces the element gathers.
    Ragged tiles, beta != 0,
    integer mode bitwise."""
    monkeypatch.setenv("TC_F32_UMMA", "1")
    monkeypatch.setenv("TC_UMMA_SHIFT", shift)
    case = W.Case("f32shift", "mab", "mkj", "abjk", lens, dtype=torch.float32, alpha=0.75,
                  beta=-0.5, c_init="dist", seed=47)
    check(case)
    case.dist = "int"
    check(case, bitwise=True)


@pytest.mark.parametrize("shift", ["2", "0"], ids=["shifted", "elements"])
def test_f32_shifted_n_vectors_guard(shift, monkeypatch):
    """Mode 12 over-fetches up to 3 floats on either side of every run: B lives in a NaN-filled,
    16-byte aligned buffer with NaN gaps between its runs and between its K slices, so a value
    picked from the wrong place of a slot poisons C; C must stay finite and match the oracle."""
    monkeypatch.setenv("TC_F32_UMMA", "1")
    monkeypatch.setenv("TC_UMMA_SHIFT", shift)
    lens = dict(m=260, a=21, b=19, k=5, j=7)
    case = W.Case("f32shiftg", "mab", "mkj", "abjk", lens, dtype=torch.float32, alpha=1.0,
                  beta=0.5, c_init="dist", seed=53)
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    sa, sb = 1, 21 + 2                  # two NaNs after every run of a
    sj = sb * 19 + 3
    sk = sj * 7 + 1
    buf = torch.full((sk * 5 + 64,), float("nan"), device="cuda")
    assert buf.data_ptr() % 16 == 0
    Bd = buf.as_strided((21, 19, 7, 5), (sa, sb, sj, sk), 4)   # 16-byte aligned base
    Bd.copy_(B.cuda())
    Cd = C.cuda()
    tc().contract(case.spec, A.cuda(), Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    got = Cd.cpu()
    assert torch.isfinite(got).all()
    assert relerr(got.numpy(), ref.numpy()) <= 1e-5


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.usefixtures("both_small_paths")
def test_f32_misaligned_views():
    g = torch.Generator().manual_seed(4)
    bigA = torch.rand(70, 9, 61, generator=g)
    bigB = torch.rand(61, 5, 50, generator=g)
    bigC = torch.rand(71, 53, generator=g)
    for off in (0, 1, 2, 3):
        A = bigA[off:off + 65, 3, :57]
        B = bigB[:57, 2, off:off + 47]
        C = bigC[off:off + 65, 1:48]
        ref = C.clone()
        oracle.contract("mn-mk-kn", A, B, ref, 1.0, -1.0)
        Cd = bigC.cuda()[off:off + 65, 1:48]
        tc().contract("mn-mk-kn", bigA.cuda()[off:off + 65, 3, :57],
                      bigB.cuda()[:57, 2, off:off + 47], Cd, 1.0, -1.0)
        assert relerr(Cd.cpu().numpy(), ref.numpy()) < 1e-6


# ---------------------------------------------------------------------------------------------
# persistent schedule: data-parallel waves + stream-K tail
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("mnk", [(100, 120, 20000), (128, 128, 4096), (1000, 1200, 700),
                                 (128 * 12, 128 * 13, 2000), (2048, 2048, 64)])
@pytest.mark.parametrize("beta", [0.0, 0.75])
def test_stream_k_splits(mnk, beta):
    """Single tiles with long K (up to 16 pieces per tile), partial waves, 156 tiles (one wave
    plus 8), and a short K; beta != 0 exercises the ordered fix-up of the first piece."""
    case = W.Case("sk", "mn", "mk", "kn", dict(zip("mnk", mnk)), alpha=0.5, beta=beta,
                  c_init="dist", seed=31)
    check(case)
    case.dist = "int"
    check(case, bitwise=True)


@pytest.mark.parametrize("weights", ["1", "0"])
@pytest.mark.parametrize("mnk", [(323, 323, 30000), (200, 300, 20000), (129, 1000, 9000),
                                 (1000, 70, 5000), (300, 3000, 4000)])
@pytest.mark.parametrize("beta", [0.0, 0.75])
def test_stream_k_work_weights(mnk, beta, weights, monkeypatch):
    """Ragged few-tile shapes (every tile in the stream-K tail, edge tiles skipping empty MMAs):
    the work-weighted split (Sched::weighted, TC_SK_WEIGHTS) gives edge tiles' CTAs more K
    iterations; results bitwise equal to the oracle's on integer inputs either way (the
    ordered fix-up is unchanged, only the piece boundaries move)."""
    monkeypatch.setenv("TC_SK_WEIGHTS", weights)
    case = W.Case("skw", "mn", "mk", "kn", dict(zip("mnk", mnk)), alpha=0.5, beta=beta,
                  dist="int", c_init="dist", seed=35)
    check(case, bitwise=True)


@pytest.mark.parametrize("csk", ["0", "8", "16", "pow2"])
@pytest.mark.parametrize("mnk", [(512, 512, 512), (323, 323, 3000), (200, 700, 1000),
                                 (1024, 1024, 600), (130, 129, 70), (640, 640, 640),
                                 (512, 640, 768), (500, 380, 900)])
@pytest.mark.parametrize("beta", [0.0, 0.75])
def test_cluster_split_k(mnk, beta, csk, monkeypatch):
    """Few-tile fp64 shapes through cluster split-K (Sched::csplit: S CTAs of a cluster share a
    tile's K loop, partials summed in rank order through distributed shared memory; S up to 8,
    or 16 non-portable with TC_CSK_MAX=16; sizes 5-7, whose row shares of the 128-row tile are
    uneven, unless TC_CSK_POW2=1) and through the stream-K fix-up chain (TC_CSK=0):
    bitwise equal to the oracle on integer inputs, ragged edges, beta != 0, both C layouts."""
    monkeypatch.setenv("TC_CSK", "0" if csk == "0" else "1")
    monkeypatch.setenv("TC_CSK_POW2", "1" if csk == "pow2" else "0")
    monkeypatch.setenv("TC_CSK_MAX", "16" if csk == "16" else "8")
    m, n, k = mnk
    for spec in ("mn-mk-kn", "nm-km-nk"):
        lc, la, lb = spec.split("-")
        case = W.Case("csk_" + spec, lc, la, lb, {"m": m, "n": n, "k": k}, alpha=0.5, beta=beta,
                      dist="int", c_init="dist", seed=57)
        check(case, bitwise=True)


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("mnk", [(100, 120, 20000), (1000, 1200, 700), (128 * 12, 128 * 13, 2000),
                                 (2366, 1012, 1935)])
@pytest.mark.parametrize("beta", [0.0, 0.75])
def test_stream_k_splits_f32(mnk, beta):
    """The fp32 kernels' stream-K pieces (fix-up order, beta on the first piece); integer-valued
    inputs make every partial sum exact, so the split result must match bit for bit."""
    case = W.Case("skf", "mn", "mk", "kn", dict(zip("mnk", mnk)), alpha=0.5, beta=beta,
                  c_init="dist", seed=33, dtype=torch.float32)
    check(case)
    case.dist = "int"
    check(case, bitwise=True)


@pytest.mark.usefixtures("both_f32_paths")
@pytest.mark.parametrize("k", [1024, 16384])
def test_f32_one_signed_bias(k):
    """One-signed data (U[0, 1)) lets accumulation biases add up instead of cancelling; the
    tcgen05 kernel's chunked accumulation (R18) keeps the error K-independent, measured
    7.6e-7 (profiles/r01/ab_umma_chunk.txt). Bound: the 1e-5 tolerance with a 5x margin."""
    g = torch.Generator(device="cuda").manual_seed(k)
    A = torch.rand(256, k, device="cuda", generator=g)
    B = torch.rand(k, 192, device="cuda", generator=g)
    C = torch.empty(256, 192, device="cuda")
    tc().contract("mn-mk-kn", A, B, C)
    ref = A.double() @ B.double()
    assert ((C.double() - ref).norm() / ref.norm()).item() < 2e-6


@pytest.mark.usefixtures("both_f32_paths")
def test_stream_k_deterministic_f32():
    case = W.Case("skdf", "mn", "mk", "kn", {"m": 2366, "n": 1012, "k": 1935}, alpha=1.0,
                  beta=0.5, c_init="dist", seed=34, dtype=torch.float32)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    outs = []
    for _ in range(3):
        C = Cd.clone()
        tc().contract(case.spec, Ad, Bd, C, case.alpha, case.beta)
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    ref = case.alpha * (Ad.double() @ Bd.double()) + case.beta * Cd.double()
    assert relerr(outs[0].cpu().numpy(), ref.cpu().numpy()) < 1e-5


def test_stream_k_deterministic_and_matches_data_parallel():
    case = W.Case("skd", "mn", "mk", "kn", {"m": 1900, "n": 1700, "k": 3000}, alpha=1.0,
                  beta=0.5, c_init="dist", seed=32)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    outs = []
    for _ in range(3):
        C = Cd.clone()
        tc().contract(case.spec, Ad, Bd, C, case.alpha, case.beta)
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    ref = case.alpha * (Ad @ Bd) + case.beta * Cd
    assert relerr(outs[0].cpu().numpy(), ref.cpu().numpy()) < 1e-12


# ---------------------------------------------------------------------------------------------
# §8(f) follow-on families: f2 = the paper's 24 fig:bench index strings (synthetic sizes),
# f1 = rank-k updates (m = n = 16000, k = 5..500)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("idx", range(24))
def test_f2_fig_bench_scaled_full(idx):
    case = W.fig_bench(idx, elems=2 ** 12)
    case.c_init, case.beta = "dist", -0.5
    check(case)


@pytest.mark.parametrize("idx", range(24))
def test_f2_fig_bench_full_sampled(idx):
    case = W.fig_bench(idx)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=2, seed=idx)
    assert torch.isfinite(c1).all()
    assert e < 1e-12


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("lens", [{"a": 40, "b": 36, "c": 67, "d": 130},
                                  {"a": 33, "b": 50, "c": 67, "d": 71},
                                  {"a": 130, "b": 129, "c": 323, "d": 66}])
def test_subdivision_with_remainder(lens, dtype):
    """fig:bench's ab-cad-dcb class (A and B have different unit-stride dimensions in P) with
    lengths that have no power-of-two divisor <= 4: the device entry point runs the divisible
    main part of the label (sub-divided) and the remainder, possibly twice (both labels); beta
    applies once. Bitwise with integer inputs."""
    case = W.Case("subrem", "ab", "cad", "dcb", lens, dtype=dtype, alpha=0.5, beta=-0.75,
                  c_init="dist", seed=61)
    check(case)
    case.dist = "int"
    check(case, bitwise=True)


@pytest.fixture(params=["1", "0"], ids=["rankk", "tile"])
def both_rankk_paths(request, monkeypatch):
    """K <= 16 contractions with large free extents through the rank-k kernel (rankk.cu) and,
    with TC_RANKK=0, through the tile kernels; the library reads TC_RANKK on every call."""
    monkeypatch.setenv("TC_RANKK", request.param)
    return request.param


@pytest.mark.usefixtures("both_rankk_paths")
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("mnk", [(2048, 2048, 5), (2100, 1037, 8), (4096, 1024, 1)])
def test_rankk_kernel_shapes(mnk, dtype):
    """Rank-k shapes (ragged column blocks, K = 1, 5, 8), beta != 0, both layouts, so that
    C's unit stride sits in either free bundle (the kernel takes only C-rows-contiguous ones)."""
    m, n, k = mnk
    for spec in ("mn-mk-kn", "nm-km-nk"):
        lc, la, lb = spec.split("-")
        case = W.Case("rk_" + spec, lc, la, lb, {"m": m, "n": n, "k": k}, dtype=dtype,
                      alpha=0.5, beta=-0.25, c_init="dist", seed=51)
        Ad, Bd, Cd = W.make_tensors(case, "cuda")
        C0 = Cd.clone()
        tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
        e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=6, seed=k)
        assert torch.isfinite(c1).all()
        assert e < TOL[dtype]


@pytest.mark.usefixtures("both_rankk_paths")
@pytest.mark.parametrize("i", range(7))
def test_f1_rankk_full_sampled(i):
    case = W.rankk(i)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    e, c1, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=3, seed=i)
    assert torch.isfinite(c1).all()
    assert e < 1e-12
    del Ad, Bd, Cd, C0
    torch.cuda.empty_cache()


@pytest.mark.parametrize("i", range(7))
def test_f1_rankk_scaled_full(i):
    case = W.rankk(i, mn=300)
    check(case)


# ---------------------------------------------------------------------------------------------
# guard bands (compute-sanitizer is closed on this pool): operands live inside NaN-filled
# buffers, so reading any element outside an operand's index space poisons C; C lives inside a
# sentinel-filled buffer whose untouched bytes must survive bitwise.
# ---------------------------------------------------------------------------------------------

def _embed(t, device, fill, rs, gap):
    """Copy tensor t into a larger buffer (filled with `fill`) with random extra stride gaps and
    a random offset; return the strided view."""
    lens = list(t.shape)
    order = list(rs.permutation(len(lens)))
    strides, s = [0] * len(lens), 1
    for d in order:
        strides[d] = s
        s *= lens[d] + int(rs.randint(0, gap + 1))
    off = int(rs.randint(0, 5))
    buf = torch.full((off + s + int(rs.randint(0, 9)),), fill, dtype=t.dtype, device=device)
    view = buf.as_strided(lens, strides, off)
    view.copy_(t.to(device))
    return buf, view


@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_guard_bands(seed, dtype):
    rs = np.random.RandomState(1000 + seed)
    case = W.random_tiny_case(seed, max_rank=6, max_len=9, dtype=dtype)
    if seed % 3 == 0:   # a few larger ones: several tiles, stream-K pieces, ragged tails
        case = W.cfg4(seed % 20, dtype)
        case = case.scaled({x: max(2, min(n, int(round(n ** 0.55)))) for x, n in case.lens.items()})
        case.beta, case.c_init = 0.5, "dist"
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    bufA, Ad = _embed(A, "cuda", float("nan"), rs, 3)
    bufB, Bd = _embed(B, "cuda", float("nan"), rs, 3)
    bufC, Cd = _embed(C, "cuda", 12345.0, rs, 3)
    mask = torch.ones(bufC.numel(), dtype=torch.bool, device="cuda")
    mask.as_strided(Cd.shape, Cd.stride(), Cd.storage_offset()).fill_(False)
    before = bufC[mask].clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    assert torch.equal(bufC[mask], before), "write outside C"
    got = Cd.cpu()
    assert torch.isfinite(got).all() or not torch.isfinite(ref).all(), "read outside A/B"
    assert relerr(got.numpy(), ref.numpy()) <= TOL[dtype]


@pytest.mark.parametrize("form", ["128", "256", "pair"])
@pytest.mark.parametrize("seed", [0, 3, 6, 9])
def test_guard_bands_f32_forms(seed, form, monkeypatch):
    """Guard bands for every form of the fp32 tcgen05 kernel on scaled cfg4 cases (several tiles,
    stream-K pieces, ragged tails)."""
    monkeypatch.setenv("TC_F32_UMMA", "1")
    monkeypatch.setenv("TC_UMMA_FORM", form)
    test_guard_bands(seed, torch.float32)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("spec", ["mn-mk-kn", "nm-km-nk"])
def test_guard_bands_rankk(spec, dtype):
    """Guard bands around a rank-k contraction (rankk.cu, both row mappings)."""
    rs = np.random.RandomState(77)
    lc, la, lb = spec.split("-")
    case = W.Case("rkguard", lc, la, lb, {"m": 2050, "n": 2049, "k": 5}, dtype=dtype,
                  alpha=0.5, beta=0.25, c_init="dist", seed=78)
    A, B, C = W.make_tensors(case, "cpu")
    bufA, Ad = _embed(A, "cuda", float("nan"), rs, 2)
    bufB, Bd = _embed(B, "cuda", float("nan"), rs, 2)
    bufC, Cd = _embed(C, "cuda", 12345.0, rs, 2)
    mask = torch.ones(bufC.numel(), dtype=torch.bool, device="cuda")
    mask.as_strided(Cd.shape, Cd.stride(), Cd.storage_offset()).fill_(False)
    before = bufC[mask].clone()
    C0 = Cd.clone()
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    assert torch.equal(bufC[mask], before), "write outside C"
    assert torch.isfinite(Cd).all(), "read outside A/B"
    e, _, _ = sampled_check(case, Ad, Bd, C0, Cd, per_label=8, seed=5)
    assert e < TOL[dtype]


# ---------------------------------------------------------------------------------------------
# skinny contractions (skinny.cu: fp64, K <= 80, one free extent <= 96, the other >= 4096)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("spec,lens,beta", [
    ("mn-mk-kn", {"m": 5000, "n": 37, "k": 29}, 0.5),      # X = A along its rows
    ("mn-km-kn", {"m": 4100, "n": 96, "k": 80}, 0.0),      # X = A along K (transposing gather)
    ("mn-mk-kn", {"m": 50, "n": 6000, "k": 13}, -1.0),     # small M: X = B, along K
    ("mn-mk-nk", {"m": 64, "n": 4097, "k": 80}, 0.0),      # small M: X = B along its rows
    ("mn-mk-kn", {"m": 4096, "n": 1, "k": 1}, 1.0),        # degenerate N = K = 1
    ("abcde-efbad-cf", {"a": 9, "b": 9, "c": 19, "d": 9, "e": 9, "f": 23}, 0.0),  # fig:bench 0
])
@pytest.mark.parametrize("skinny", ["1", "0", ""])
def test_skinny_shapes(spec, lens, beta, skinny, monkeypatch):
    monkeypatch.setenv("TC_SKINNY", skinny)   # the library reads it on every call
    lc, la, lb = spec.split("-")
    case = W.Case("skinny_" + spec, lc, la, lb, lens, alpha=0.75, beta=beta,
                  c_init="dist" if beta else "nan", seed=31)
    check(case)
    case.dist, case.alpha = "int", 2.0
    case.beta = 0.5 if beta else 0.0
    check(case, bitwise=True)


@pytest.mark.parametrize("spec,lens", [
    ("mn-mk-kn", {"m": 7001, "n": 32, "k": 32}),       # X = A along its rows, NP = KP = 32
    ("mn-km-kn", {"m": 4099, "n": 17, "k": 9}),        # X = A along K, NP = 32, KP = 12
    ("mn-mk-nk", {"m": 5, "n": 9000, "k": 31}),        # small M: X = B along its rows, NP = 16
    ("mn-mk-kn", {"m": 3, "n": 5000, "k": 2}),         # small M: X = B along K
    ("abcde-efbad-cf", {"a": 16, "b": 7, "c": 32, "d": 11, "e": 24, "f": 32}),   # sub-divided
    ("mn-mk-kn", {"m": 300000, "n": 32, "k": 32}),     # many blocks per CTA (ring wraps)
    ("mn-mk-kn", {"m": 70001, "n": 76, "k": 76}),      # Y fragments from shared memory, NP = 80
    ("mn-km-kn", {"m": 4099, "n": 96, "k": 80}),       # largest resident operand, X along K
    ("abcd-dbea-ec", {"a": 16, "b": 12, "c": 40, "d": 24, "e": 36}),   # fig:bench 2, sub-divided
])
@pytest.mark.parametrize("ws", ["0", "cg1", "cg2", "st2", "st3", "big0"])
def test_skinny_warp_specialised(spec, lens, ws, monkeypatch):
    """The skinny kernel's warp-specialised form: producer warps fill an S-deep ring tracked by
    mbarriers, 1 or 2 consumer groups multiply (Y in registers for NP, KP <= 32, else from
    shared memory) and store; against the synchronous form (ws = 0, big0 for the larger resident
    operands) and the oracle, bitwise on integer inputs, beta = 0 and beta != 0."""
    monkeypatch.setenv("TC_SKINNY_WS", "0" if ws == "0" else "1")
    monkeypatch.setenv("TC_SKINNY_WS_CG", "1" if ws == "cg1" else "2")
    monkeypatch.setenv("TC_SKINNY_WS_STAGES", ws[2:] if ws.startswith("st") else "0")
    monkeypatch.setenv("TC_SKINNY_WS_BIG", "0" if ws == "big0" else "1")
    lc, la, lb = spec.split("-")
    for beta in (0.0, 0.5):
        case = W.Case("skinny_ws_" + spec, lc, la, lb, lens, alpha=2.0, beta=beta, dist="int",
                      c_init="dist" if beta else "nan", seed=41)
        check(case, bitwise=True)


@pytest.mark.parametrize("shift", [0, 1, 2])
def test_skinny_offset_views(shift):
    """The skinny kernel on an X viewed at an element offset (8-byte and 16-byte shifted bases),
    ragged rows: bitwise equal to the oracle (integer inputs)."""
    m, n, k = 5003, 32, 32
    g = torch.Generator().manual_seed(7 + shift)
    big = torch.randint(-8, 9, (m * k + 8,), generator=g).double()
    A = big[shift:shift + m * k].view(k, m).t()          # column-major (m contiguous), offset
    B = torch.randint(-8, 9, (k, n), generator=g).double()
    C0 = torch.randint(-8, 9, (m, n), generator=g).double()
    ref = C0.clone()
    oracle.contract("mn-mk-kn", A, B, ref, 2.0, 0.5)
    bigd = big.cuda()
    Ad = bigd[shift:shift + m * k].view(k, m).t()
    Cd = C0.cuda()
    tc().contract("mn-mk-kn", Ad, B.cuda(), Cd, 2.0, 0.5)
    assert torch.equal(Cd.cpu(), ref)


@pytest.mark.parametrize("lens", [
    {"a": 16, "b": 7, "c": 32, "d": 11, "e": 24, "f": 20},   # bu = bv = 8: skew 2
    {"a": 12, "b": 9, "c": 17, "d": 13, "e": 8, "f": 33},    # bu = 8, bv = 4: skew 2
    {"a": 8, "b": 10, "c": 40, "d": 9, "e": 12, "f": 8},     # bu = 4, bv = 8: skew 4
])
@pytest.mark.parametrize("sw", ["", "0", "1", "3"])
def test_skinny_ring_skew(lens, sw, monkeypatch):
    """The skinny kernel's skewed X ring (block row r at r + sw (r / 16), chosen on the host from
    the sub-division (bu, bv); TC_SKINNY_SW forces one): every skew gives the oracle's result,
    bitwise on integer inputs, with a ragged last block."""
    monkeypatch.setenv("TC_SKINNY_SW", sw)
    case = W.Case("skinny_skew", "abcde", "efbad", "cf", lens, alpha=2.0, beta=0.5,
                  dist="int", c_init="dist", seed=37)
    check(case, bitwise=True)


@pytest.mark.parametrize("lens", [
    {"a": 32, "b": 5, "c": 32, "d": 7, "e": 32, "f": 32},    # bv = 16 / 32, bu = 4 / 2
    {"a": 48, "b": 3, "c": 20, "d": 9, "e": 24, "f": 12},    # bv = 16, bu = 4; ragged last block
])
@pytest.mark.parametrize("env", ["TC_SKINNY_BV=16", "TC_SKINNY_BV=32", "TC_SKINNY_BU=16",
                                 "TC_SKINNY_BU=32"])
def test_skinny_run_lengths(lens, env, monkeypatch):
    """Other run lengths in the skinny sub-division (TC_SKINNY_BV / _BU: C's or X's runs up to 16
    or 32 elements, the other's capped at 64 / that): bitwise the oracle's result on integer
    inputs, alpha and beta != 0."""
    name, val = env.split("=")
    monkeypatch.setenv(name, val)   # part of the plan-cache key
    case = W.Case("skinny_bv", "abcde", "efbad", "cf", lens, alpha=2.0, beta=0.5,
                  dist="int", c_init="dist", seed=41)
    check(case, bitwise=True)


# ---------------------------------------------------------------------------------------------
# negative strides (accepted for A, B and C by the C ABI, reading R7) through the raw binding
# ---------------------------------------------------------------------------------------------

def _reversed_desc(t_dev, labels, flip):
    """Descriptor of the device tensor t_dev walked backwards along the dims in `flip`: the
    data pointer moves to the last element of each flipped dim and its stride changes sign."""
    lens, strides = list(t_dev.shape), list(t_dev.stride())
    off = 0
    for d in flip:
        off += (lens[d] - 1) * strides[d]
        strides[d] = -strides[d]
    ptr = t_dev.data_ptr() + off * t_dev.element_size()
    return tc().Desc(labels, lens, strides, ptr)


@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("lens", [{"m": 300, "n": 200, "k": 150},    # tensor-core tile kernel
                                  {"m": 5000, "n": 40, "k": 30},     # skinny kernel (fp64)
                                  {"m": 33, "n": 17, "k": 9}])       # tiny kernel
def test_negative_strides(lens, dtype):
    g = torch.Generator().manual_seed(7)
    m, n, k = lens["m"], lens["n"], lens["k"]
    A = torch.randint(-4, 5, (m, k), generator=g).to(dtype)
    B = torch.randint(-4, 5, (k, n), generator=g).to(dtype)
    C = torch.randint(-4, 5, (m, n), generator=g).to(dtype)
    # reference: A read backwards along m, B backwards along k, C written backwards along n
    Ar, Br = A.flip(0), B.flip(0)
    ref = C.flip(1).clone()
    oracle.contract("mn-mk-kn", Ar, Br, ref, 2.0, 0.5)
    Ad, Bd, Cd = A.cuda(), B.cuda(), C.cuda()
    code = tc()._dtype_code(dtype)
    tc().tc_contract(code, 2.0, _reversed_desc(Ad, "mk", [0]), _reversed_desc(Bd, "kn", [0]), 0.5,
                     _reversed_desc(Cd, "mn", [1]), None)
    torch.cuda.synchronize()
    assert torch.equal(Cd.cpu().flip(1), ref)



# ---------------------------------------------------------------------------------------------
# multi-GPU sharding on one device: every rank's shard contraction (zero-copy narrowed views,
# dist.contract_shard, the call bench.py makes per GPU) assembled = the full contraction
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_blocks_assemble_full_result(world):
    from paper_1607_00291_b200 import dist as tdist
    case = W.cfg5(12, 6)
    case.dist = "int"
    Ad, Bd, _ = W.make_tensors(case, "cuda", gen_device="cpu")
    full = W.colmajor_view(torch.full((math.prod(case.shape(case.lab_c)),), float("nan"),
                                      dtype=torch.float64, device="cuda"), case.shape(case.lab_c))
    tc().contract(case.spec, Ad, Bd, full, 1.0, 0.0)
    assembled = torch.full_like(full, float("nan"))
    for rank in range(world):
        ranges = tdist.shard_ranges(world, rank, case.lens, "abc")
        shape = tdist.shard_shape(case.lab_c, case.lens, ranges)
        Cs = W.colmajor_view(torch.empty(math.prod(shape), dtype=torch.float64, device="cuda"), shape)
        tdist.contract_shard(case.spec, Ad, Bd, Cs, ranges, 1.0, 0.0)
        tdist.narrow(assembled, case.lab_c, ranges).copy_(Cs)
    torch.cuda.synchronize()
    assert torch.equal(assembled, full)


# ---------------------------------------------------------------------------------------------
# 64-bit offsets (a tensor spanning >= 2^31 elements switches every table to int64)
# ---------------------------------------------------------------------------------------------

@pytest.mark.usefixtures("both_small_paths")
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("lens", [{"m": 128, "n": 128, "k": 160},   # tile kernel, int64 tables
                                  {"m": 5000, "n": 40, "k": 30},    # skinny kernel
                                  {"m": 20, "n": 12, "k": 30},      # tiny kernel
                                  {"m": 2048, "n": 2048, "k": 5}])  # rank-k kernel
def test_int64_offsets_large_span(lens, dtype):
    """A is a strided view whose K stride is 2^27 elements, so its address span exceeds 2^31
    elements (a 16-32 GiB buffer, untouched except where A lives). fp32 takes the FFMA2 tile
    kernel here (the tcgen05 kernel has 32-bit offsets only)."""
    m, n, k = lens["m"], lens["n"], lens["k"]
    g = torch.Generator().manual_seed(9)
    A = torch.randint(-4, 5, (m, k), generator=g).to(dtype)
    B = torch.randint(-4, 5, (k, n), generator=g).to(dtype)
    ref = torch.zeros(m, n, dtype=dtype)
    oracle.contract("mn-mk-kn", A, B, ref, 1.0, 0.0)
    stride_k = 1 << 27
    while stride_k * (k - 1) < (1 << 31):   # short K: a longer stride keeps the span > 2^31
        stride_k *= 2
    big = torch.empty(stride_k * (k - 1) + m, dtype=dtype, device="cuda")
    Ad = big.as_strided((m, k), (1, stride_k))
    Ad.copy_(A.cuda())
    Cd = torch.full((m, n), float("nan"), dtype=dtype, device="cuda")
    info = tc().Plan.for_tensors("mn-mk-kn", Ad, B.cuda(), Cd).info()
    assert info["idx64"]
    tc().contract("mn-mk-kn", Ad, B.cuda(), Cd, 1.0, 0.0)
    torch.cuda.synchronize()
    assert torch.equal(Cd.cpu(), ref)
    del big
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("alpha,beta", [(1.5, 0.0), (0.0, 0.5), (-1.0, 2.0)])
def test_host_path_dtypes_and_scalars(dtype, alpha, beta):
    """tc_contract_host on both element types; alpha = 0 uploads only C (R1)."""
    case = W.cfg3(True, v=48, o=24)       # 48 MB operands: chunked along C's outer label
    case.dtype, case.dist, case.alpha, case.beta, case.c_init = dtype, "int", alpha, beta, "dist"
    A, B, C = W.make_tensors(case, "cpu")
    if alpha == 0.0:
        A.fill_(float("nan")); B.fill_(float("nan"))
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, alpha, beta)
    Cp = C.clone().pin_memory()
    tc().contract_host(case.spec, A.pin_memory(), B.pin_memory(), Cp, alpha, beta)
    assert torch.equal(Cp, ref)
