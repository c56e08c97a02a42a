"""GPU robustness of the C ABI and the launch machinery:

  * the first call of a new plan on a fresh non-blocking stream (tables and stream-K flags are
    created on the legacy stream and must be complete before any stream reads them);
  * stream-K flags tagged with a per-launch epoch: hundreds of back-to-back split launches on
    several streams stay bitwise deterministic (no reset between launches);
  * tc_plan_execute's alias check, dtype / device checks of the binding;
  * the fp32 3xTF32 split (reading R18) on operands whose magnitudes span 2^-40 .. 2^40.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_00291_b200  # noqa: F401


def tc():
    import paper_1607_00291_b200 as m
    return m


def _int_case(m, n, k, dtype=torch.float64, beta=0.5, seed=3):
    return W.Case("rb", "mn", "mk", "kn", {"m": m, "n": n, "k": k}, dtype=dtype, dist="int",
                  alpha=2.0, beta=beta, c_init="dist", seed=seed)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_first_call_on_fresh_nonblocking_stream(dtype):
    """A never-seen plan (odd shape), first launched on a brand-new non-blocking stream, with a
    stream-K tail (K long, tiles < #SMs): bitwise equal to the oracle (integer inputs)."""
    m, n, k = (1000 + 7 * (dtype == torch.float32), 1101, 3333)
    case = _int_case(m, n, k, dtype)
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Ad, Bd, Cd = A.cuda(), B.cuda(), C.cuda()
        tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    s.synchronize()
    assert torch.equal(Cd.cpu(), ref)


@pytest.mark.parametrize("form", ["f64", "umma", "ffma", "pair"])
def test_epoch_tagged_flags_many_launches(form, monkeypatch):
    """300 launches with stream-K pieces, alternating over three streams, reusing each stream's
    flag buffer without resets: every result bitwise equal to the first."""
    dtype = torch.float64 if form == "f64" else torch.float32
    if form == "ffma":
        monkeypatch.setenv("TC_F32_UMMA", "0")
    if form == "pair":
        monkeypatch.setenv("TC_UMMA_FORM", "pair")
    case = _int_case(700, 650, 4000, dtype, beta=0.25, seed=8)
    Ad, Bd, Cd = W.make_tensors(case, "cuda")
    ref = Cd.clone()
    tc().contract(case.spec, Ad, Bd, ref, case.alpha, case.beta)
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = [Cd.clone() for _ in range(6)]
    torch.cuda.synchronize()
    for i in range(300):
        s = streams[i % 3]
        with torch.cuda.stream(s):
            o = outs[i % 6]
            o.copy_(Cd)
            tc().contract(case.spec, Ad, Bd, o, case.alpha, case.beta)
        if i % 6 == 5:
            torch.cuda.synchronize()
            for o in outs:
                assert torch.equal(o, ref), i
    torch.cuda.synchronize()


def test_plan_execute_alias_check():
    A = torch.randn(64, 64, dtype=torch.float64, device="cuda")
    B = torch.randn(64, 64, dtype=torch.float64, device="cuda")
    C = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    p = tc().Plan.for_tensors("mn-mk-kn", A, B, C)
    p.execute(A, B, C)
    torch.cuda.synchronize()
    assert torch.allclose(C, A @ B, rtol=1e-12, atol=1e-12)
    with pytest.raises(tc().TCError) as ei:
        p.execute(A, B, A)                 # C is A
    assert ei.value.code == 4
    big = torch.zeros(64 * 64 + 32, dtype=torch.float64, device="cuda")
    Cv = big[32:].view(64, 64)
    Bv = big[:64 * 64].view(64, 64)        # overlaps C's first 64*64 - 32 elements
    with pytest.raises(tc().TCError) as ei:
        p.execute(A, Bv, Cv)
    assert ei.value.code == 4


def test_binding_rejects_mixed_dtypes_and_devices():
    A = torch.randn(8, 8, dtype=torch.float32, device="cuda")
    B = torch.randn(8, 8, dtype=torch.float64, device="cuda")
    C = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        tc().contract("mn-mk-kn", A, B, C)
    with pytest.raises(TypeError):
        tc().contract_host("mn-mk-kn", A.cpu(), B.cpu(), C.cpu())
    with pytest.raises(ValueError):
        tc().contract("mn-mk-kn", B.cpu(), B, C)
    with pytest.raises(ValueError):
        tc().contract_host("mn-mk-kn", B, B.cpu(), C.cpu())
    assert torch.equal(C, torch.zeros_like(C))


@pytest.mark.parametrize("form", ["0", "128", "256", "pair"])
@pytest.mark.parametrize("shape", [(512, 384, 1536), (300, 200, 700)])
def test_f32_wide_dynamic_range(form, shape, monkeypatch):
    """Reading R18 on operands whose rows / columns are scaled by 2^e, e uniform in [-40, 40]:
    C_ij spans 2^-80 .. 2^80. Checked against the fp64 product of the same fp32 values, per
    element against the dot-product bound: |C - ref| <= 1e-5 * (|A| |B|)_ij (the 3xTF32 split
    drops A_lo B_lo ~ 2^-22 |a||b| per term and accumulates in fp32), and normwise <= 1e-5."""
    if form == "0":
        monkeypatch.setenv("TC_F32_UMMA", "0")
    else:
        monkeypatch.setenv("TC_UMMA_FORM", form)
    m, n, k = shape
    g = torch.Generator().manual_seed(m + k)
    ea = torch.randint(-40, 41, (m, 1), generator=g).double()
    eb = torch.randint(-40, 41, (1, n), generator=g).double()
    ek = torch.randint(-6, 7, (1, k), generator=g).double()
    A = ((torch.rand(m, k, generator=g, dtype=torch.float64) * 2 - 1) * torch.exp2(ea + ek)).float()
    B = ((torch.rand(k, n, generator=g, dtype=torch.float64) * 2 - 1)
         * torch.exp2(eb - ek.t())).float()
    Ad, Bd = A.cuda(), B.cuda()
    Cd = torch.full((m, n), float("nan"), device="cuda")
    tc().contract("mn-mk-kn", Ad, Bd, Cd)
    got = Cd.cpu().double()
    ref = A.double() @ B.double()
    bound = A.double().abs() @ B.double().abs()
    assert torch.isfinite(got).all()
    ratio = ((got - ref).abs() / bound).max().item()
    assert ratio <= 1e-5, ratio
    assert ((got - ref).norm() / ref.norm()).item() <= 1e-5


def test_concurrent_host_threads_on_separate_streams():
    """Four host threads call the C ABI at once (ctypes releases the GIL), each on its own stream,
    mixing shapes that share plans with shapes that do not and stream-K splits; every result is
    bitwise equal to the single-threaded one (integer inputs)."""
    import threading
    cases = [_int_case(700, 650, 4000, torch.float64, seed=11),
             _int_case(700, 650, 4000, torch.float32, seed=12),
             _int_case(333, 1200, 2500, torch.float64, seed=13),
             _int_case(2000, 300, 700, torch.float32, seed=14)]
    tensors = [W.make_tensors(c, "cuda") for c in cases]
    refs = []
    for c, (Ad, Bd, Cd) in zip(cases, tensors):
        r = Cd.clone()
        tc().contract(c.spec, Ad, Bd, r, c.alpha, c.beta)
        refs.append(r)
    torch.cuda.synchronize()
    errors = []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for i in range(40):
                    j = (t + i) % len(cases)
                    c, (Ad, Bd, Cd) = cases[j], tensors[j]
                    out = Cd.clone()
                    tc().contract(c.spec, Ad, Bd, out, c.alpha, c.beta)
                    s.synchronize()
                    if not torch.equal(out, refs[j]):
                        errors.append((t, i, j))
        except Exception as e:   # pragma: no cover
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:5]
