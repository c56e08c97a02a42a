"""GPU parity at full BASELINE sizes, on EVERY element of C (pin p8).

The element-wise oracle cannot finish cfg3 (5.5e11 flops) or cfg5 (8.45e13) on the host, so the
CUDA result is checked whole with Freivalds' test (oracle.freivalds_check, plain C loops in
oracle/contract.c): for seeded x over the J labels, C_new·x = alpha·A·(B·x) + beta·C_old·x
in the contraction's matrix form (§3, §6.1).

  * integer mode (A, B, C in [-4, 4], x in [-1024, 1024], pin p5): every partial sum on both
    sides is exact, so the comparison is bitwise; a wrong element escapes one vector with
    probability <= 1/2049, three vectors are used;
  * the BASELINE distributions: normwise residual
    ||C_new·x - alpha·A·(B·x) - beta·C_old·x|| / (|alpha|·||A||_F·||B·x|| + |beta|·||C_old·x||)
    <= 1e-12 (fp64) / 1e-5 (fp32) (BASELINE.json north_star tolerances).

Each runs in the launch configuration bench.py times (the same C-ABI call, full shapes).
cfg4 is also re-run at alpha = -0.5, beta = 0.5 with C ~ U[-1, 1], at full
size (every element, both modes, fp64 and every fp32 form) and scaled (element-wise oracle).
"""
import math

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


F32_FORMS = ["0", "1", "128", "256", "pair"]


def _set_f32_form(monkeypatch, form):
    if form == "0":
        monkeypatch.setenv("TC_F32_UMMA", "0")
    else:
        monkeypatch.setenv("TC_F32_UMMA", "1")
        if form != "1":
            monkeypatch.setenv("TC_UMMA_FORM", form)


def run_and_check(case, int_mode: bool, nvec: int = 3, seed: int = 0):
    """Generate the case on the device, run the CUDA path through the C ABI, copy A, B, C_old
    and C_new to the host and run the Freivalds check there. Returns the residual (0.0 in
    integer mode when exact)."""
    if int_mode:
        case.dist = "int"
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    C0 = Cd.cpu() if case.beta != 0.0 else None
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    Cn = Cd.cpu()
    del Cd
    A, B = Ad.cpu(), Bd.cpu()
    del Ad, Bd
    torch.cuda.empty_cache()
    assert torch.isfinite(Cn).all(), case.name
    r = oracle.freivalds_check(case.spec, A, B, Cn, C0, case.alpha, case.beta, nvec=nvec,
                               seed=seed, exact=int_mode)
    if int_mode:
        assert r == 0.0, (case.name, r)
    else:
        assert r <= TOL[case.dtype], (case.name, r)
    return r


# ---------------------------------------------------------------------------------------------
# cfg2, cfg3 (+ variant), cfg5: every element at full size
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("int_mode", [True, False], ids=["int", "dist"])
@pytest.mark.parametrize("transposed", [False, True], ids=["NN", "TT"])
def test_cfg2_full_every_element(transposed, int_mode):
    run_and_check(W.cfg2(transposed), int_mode)


@pytest.mark.parametrize("int_mode", [True, False], ids=["int", "dist"])
@pytest.mark.parametrize("variant", [False, True], ids=["abij", "aibj"])
def test_cfg3_full_every_element(variant, int_mode):
    run_and_check(W.cfg3(variant), int_mode)


@pytest.mark.slow
@pytest.mark.parametrize("int_mode", [True, False], ids=["int", "dist"])
def test_cfg5_full_every_element(int_mode):
    """cfg5 at full size (55296 x 27648 x 27648, 30.6 GB of operands), the bench workload."""
    run_and_check(W.cfg5(), int_mode)


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4, 8])
def test_cfg5_full_every_shard(world):
    """Every rank's shard of full-size cfg5 (C over free blocks of (a, b, c), dist.contract_shard:
    the call bench.py makes per GPU), each checked on every element against its own A/B sub-views
    (P:582-591), integer mode (exact)."""
    from paper_1607_00291_b200 import dist as tdist
    case = W.cfg5()
    case.dist = "int"
    Ad, Bd, _ = W.make_tensors(case, "cuda")
    A, B = Ad.cpu(), Bd.cpu()
    for rank in range(world):
        ranges = tdist.shard_ranges(world, rank, case.lens, "abc")
        shape = tdist.shard_shape(case.lab_c, case.lens, ranges)
        Cs = W.colmajor_view(torch.full((math.prod(shape),), float("nan"), dtype=torch.float64,
                                        device="cuda"), shape)
        tdist.contract_shard(case.spec, Ad, Bd, Cs, ranges, 1.0, 0.0)
        torch.cuda.synchronize()
        Ch = Cs.cpu()
        del Cs
        assert torch.isfinite(Ch).all(), (world, rank)
        r = oracle.freivalds_check(case.spec, tdist.narrow(A, case.lab_a, ranges),
                                   tdist.narrow(B, case.lab_b, ranges), Ch, None, 1.0, 0.0,
                                   nvec=3, seed=rank, exact=True)
        assert r == 0.0, (world, rank, r)
    del Ad, Bd
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------------------------
# cfg4 at alpha = -0.5, beta = 0.5, C ~ U[-1, 1] (SURVEY.md §8(d) correctness re-run)
# ---------------------------------------------------------------------------------------------

def _cfg4_ab(i, dtype):
    return W.cfg4(i, dtype, alpha=-0.5, beta=0.5, c_init="dist")


@pytest.mark.parametrize("int_mode", [True, False], ids=["int", "dist"])
@pytest.mark.parametrize("i", range(20))
def test_cfg4_alpha_beta_full_every_element_f64(i, int_mode):
    run_and_check(_cfg4_ab(i, torch.float64), int_mode, seed=i)


@pytest.mark.parametrize("form", F32_FORMS, ids=["ffma", "umma", "umma128", "umma256", "pair"])
@pytest.mark.parametrize("int_mode", [True, False], ids=["int", "dist"])
@pytest.mark.parametrize("i", range(20))
def test_cfg4_alpha_beta_full_every_element_f32(i, int_mode, form, monkeypatch):
    _set_f32_form(monkeypatch, form)
    run_and_check(_cfg4_ab(i, torch.float32), int_mode, seed=i)


def _scaled(case):
    lens = {x: (max(2, int(round(n ** 0.6))) if n > 64 else max(2, n // 3))
            for x, n in case.lens.items()}
    return case.scaled(lens)


def _elementwise(case):
    A, B, C = W.make_tensors(case, "cpu")
    Ad, Bd, Cd = W.make_tensors(case, "cuda", gen_device="cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    return Cd.cpu(), ref


@pytest.mark.parametrize("i", range(20))
def test_cfg4_alpha_beta_scaled_elementwise_f64(i):
    got, ref = _elementwise(_scaled(_cfg4_ab(i, torch.float64)))
    e = float((got - ref).norm() / ref.norm())
    assert e <= TOL[torch.float64], e
    case = _scaled(_cfg4_ab(i, torch.float64))
    case.dist = "int"
    got, ref = _elementwise(case)
    assert torch.equal(got, ref)


@pytest.mark.parametrize("form", F32_FORMS, ids=["ffma", "umma", "umma128", "umma256", "pair"])
@pytest.mark.parametrize("i", range(20))
def test_cfg4_alpha_beta_scaled_elementwise_f32(i, form, monkeypatch):
    _set_f32_form(monkeypatch, form)
    got, ref = _elementwise(_scaled(_cfg4_ab(i, torch.float32)))
    e = float((got.double() - ref.double()).norm() / ref.double().norm())
    assert e <= TOL[torch.float32], e
    case = _scaled(_cfg4_ab(i, torch.float32))
    case.dist = "int"
    got, ref = _elementwise(case)
    assert torch.equal(got, ref)


# ---------------------------------------------------------------------------------------------
# §8(f) families at full size, every element (integer mode)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("idx", range(24))
def test_f2_fig_bench_full_every_element(idx):
    case = W.fig_bench(idx)
    case.c_init, case.beta, case.alpha = "dist", 0.5, -1.0
    run_and_check(case, True, seed=idx)


@pytest.mark.parametrize("i", range(7))
def test_f1_rankk_full_every_element(i):
    case = W.rankk(i)
    case.c_init, case.beta = "dist", -0.5
    run_and_check(case, True, seed=i)
