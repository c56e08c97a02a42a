"""Parity of the loader ablations (§8(f) f3; pin p3(vii): forcing each loader path gives the same
result).

TC_FORCE_PATH=scatter is the paper's SMTC: every element of A and B is gathered
individually through the scatter vectors, no block-scatter fast path. TC_FORCE_PATH=blockscatter
forces the per-vector block-scatter check wherever an operand is not proven
all-vector. The library reads the variable on every call, so one process runs every path.
Integer inputs (pin p5) make all of them bitwise equal to the oracle.
"""
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


PATHS = ["", "scatter", "blockscatter"]


def _run(case, path, monkeypatch):
    if path:
        monkeypatch.setenv("TC_FORCE_PATH", path)
    else:
        monkeypatch.delenv("TC_FORCE_PATH", raising=False)
    Ad, Bd, Cd = W.make_tensors(case, "cuda", gen_device="cpu")
    tc().contract(case.spec, Ad, Bd, Cd, case.alpha, case.beta)
    torch.cuda.synchronize()
    return Cd.cpu()


def _oracle(case):
    A, B, C = W.make_tensors(case, "cpu")
    ref = C.clone()
    oracle.contract(case.spec, A, B, ref, case.alpha, case.beta)
    return ref


def _structures():
    out = [W.cfg1(), W.cfg2(False, n=300), W.cfg2(True, n=300), W.cfg3(False, v=24, o=10),
           W.cfg3(True, v=24, o=10), W.cfg5(big=12, small=6)]
    for i in (0, 3, 7, 9, 13, 15, 16, 19):
        c = W.cfg4(i)
        out.append(c.scaled({x: (max(2, int(round(n ** 0.6))) if n > 64 else max(2, n // 3))
                             for x, n in c.lens.items()}))
    return out


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("path", PATHS, ids=["default", "smtc", "blockscatter"])
@pytest.mark.parametrize("k", range(14))
def test_forced_paths_baseline_structures(k, path, dtype, monkeypatch):
    case = _structures()[k]
    case.dist, case.dtype, case.c_init = "int", dtype, "dist"
    case.alpha, case.beta = 2.0, -0.5
    got = _run(case, path, monkeypatch)
    assert torch.equal(got, _oracle(case)), (case.name, path)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("path", PATHS, ids=["default", "smtc", "blockscatter"])
@pytest.mark.parametrize("idx", range(24))
def test_forced_paths_fig_bench(idx, path, dtype, monkeypatch):
    case = W.fig_bench(idx, elems=2 ** 14, dtype=dtype)
    case.dist, case.c_init, case.alpha, case.beta = "int", "dist", 1.0, 0.5
    got = _run(case, path, monkeypatch)
    assert torch.equal(got, _oracle(case)), (case.name, path)


@pytest.mark.parametrize("path", ["scatter", "blockscatter"])
def test_forced_path_switches_within_one_process(path, monkeypatch):
    """The same cached plan runs the default path, the forced one and the default again."""
    case = W.cfg4(4)
    case.dist, case.c_init, case.beta = "int", "dist", 0.5
    case = case.scaled({x: (max(2, int(round(n ** 0.7))) if n > 64 else max(2, n // 2))
                        for x, n in case.lens.items()})
    ref = _oracle(case)
    for p in ("", path, ""):
        assert torch.equal(_run(case, p, monkeypatch), ref), p
