"""oracle -- TEST INFRASTRUCTURE ONLY.

The independent CPU oracle for the B200 contraction path. Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` leg may import it; the product package
(paper_1607_00291_b200/) never does, and the two share no code.

  contract(spec, A, B, C, alpha, beta)      plain C nested loops (oracle/contract.c), in place on C
  contract_at(spec, A, B, C, alpha, beta, idx)  the same definition for selected C elements only
  freivalds(spec, A, B, C_new, C_old, x)    pin p8: the matrix-form products B·x, A·(B·x), C_new·x,
                                            C_old·x for a full-tensor check of results too large
                                            for contract() (plain C loops, oracle/contract.c)
  freivalds_check(...)                      p8's exact (integer inputs) or normwise residual test
  brute(spec, A, B, C, alpha, beta)         a second, pure-Python statement (itertools over a dict
                                            of label values) used to pin contract() on tiny inputs
  plan.*                                    the integer steps a1-a4 (classification, heuristic,
                                            scatter and block-scatter vectors)

Tensors are torch CPU tensors or numpy arrays with arbitrary (numpy: also negative) strides;
the oracle reads them through their base pointer, lengths and element strides
(loc = sum idx*stride).

Parity status: contract/contract_at/brute pinned by tests/test_oracle_pins.py
(brute force, GEMM reduction, closed forms, invariants, integer exactness); plan.* pinned by the
paper's worked example (tests/golden/e1_worked_example.json) and SPEC.md's derived examples.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

from . import plan  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "contract.c")
_SO = os.path.join(_HERE, "_oracle.so")
_lib = None

I64P = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle/contract.c with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-std=c99", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        args = [ctypes.c_int, ctypes.c_double]
        for _ in range(2):
            args += [ctypes.c_void_p, ctypes.c_int, I64P, I64P, ctypes.c_char_p]
        args += [ctypes.c_double, ctypes.c_void_p, ctypes.c_int, I64P, I64P, ctypes.c_char_p]
        lib.oracle_contract.argtypes = args + [ctypes.c_int]
        lib.oracle_contract.restype = ctypes.c_int
        lib.oracle_contract_at.argtypes = args + [ctypes.c_int64, I64P,
                                                  ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        lib.oracle_contract_at.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        targs = []
        for _ in range(3):
            targs += [ctypes.c_void_p, ctypes.c_int, I64P, I64P, ctypes.c_char_p]
        lib.oracle_freivalds_dims.argtypes = [a for a in targs if a is not ctypes.c_void_p] + [I64P]
        lib.oracle_freivalds_dims.restype = ctypes.c_int
        DP = ctypes.POINTER(ctypes.c_double)
        lib.oracle_freivalds.argtypes = [ctypes.c_int] + targs + [ctypes.c_void_p, I64P] + \
            [DP] * 5 + [ctypes.c_int]
        lib.oracle_freivalds.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _view(t):
    """(pointer, lens, element strides, dtype code) of a torch CPU tensor or numpy array."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            assert t.device.type == "cpu", "oracle reads host memory only"
            code = {torch.float64: 0, torch.float32: 1}[t.dtype]
            return t.data_ptr(), list(t.shape), list(t.stride()), code
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(t)
    code = {np.dtype(np.float64): 0, np.dtype(np.float32): 1}[a.dtype]
    strides = [s // a.itemsize for s in a.strides]
    return a.__array_interface__["data"][0], list(a.shape), strides, code


def _arr(xs):
    a = (ctypes.c_int64 * max(len(xs), 1))(*[int(x) for x in xs])
    return a


ERRORS = {1: "rank too large", 2: "label error", 3: "shape error", 4: "out of host memory"}


def _parse(spec: str):
    parts = spec.split("-")
    if len(parts) != 3:
        raise ValueError(f"index string must be C-A-B (P:1327-1329), got {spec!r}")
    return parts[0], parts[1], parts[2]


def _args(spec, A, B, C):
    lab_c, lab_a, lab_b = _parse(spec)
    out, dts, keep = [], [], []
    for t, lab in ((A, lab_a), (B, lab_b), (C, lab_c)):
        p, lens, strides, code = _view(t)
        if len(lens) != len(lab):
            raise ValueError(f"rank of tensor ({len(lens)}) != len({lab!r})")
        la, sa = _arr(lens), _arr(strides)
        keep += [la, sa]
        out.append((ctypes.c_void_p(p), len(lens), la, sa, lab.encode()))
        dts.append(code)
    if len(set(dts)) != 1:
        raise ValueError("A, B, C must share one dtype")
    return out, dts[0], keep


def contract(spec: str, A, B, C, alpha: float = 1.0, beta: float = 0.0,
             threads: Optional[int] = None):
    """C := alpha * sum_P A*B + beta*C, in place (oracle/contract.c)."""
    (a, b, c), code, _keep = _args(spec, A, B, C)
    err = _load().oracle_contract(code, float(alpha), *a, *b, float(beta), *c, int(threads or 0))
    if err:
        raise ValueError(f"oracle: {ERRORS.get(err, err)} for {spec!r}")
    return C


def contract_at(spec: str, A, B, C, alpha: float, beta: float, idx: np.ndarray,
                threads: Optional[int] = None) -> np.ndarray:
    """alpha * sum_P A*B + beta*C_old at the C multi-indices idx[n, rank(C)] (C untouched)."""
    (a, b, c), code, _keep = _args(spec, A, B, C)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n = idx.shape[0]
    out = np.empty(n, dtype=np.float64)
    err = _load().oracle_contract_at(code, float(alpha), *a, *b, float(beta), *c, n,
                                     idx.ctypes.data_as(I64P),
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     int(threads or 0))
    if err:
        raise ValueError(f"oracle: {ERRORS.get(err, err)} for {spec!r}")
    return out


def brute(spec: str, A, B, C, alpha: float = 1.0, beta: float = 0.0) -> np.ndarray:
    """Second, independent statement of P:278-281 for tiny inputs: loop over every assignment
    of values to all labels (itertools.product over a dict), accumulate A*B into the C entry
    the assignment names. Returns the new C as a float64 numpy array in C's shape (C untouched)."""
    lab_c, lab_a, lab_b = _parse(spec)
    a, b, c = (np.asarray(x, dtype=np.float64) for x in (A, B, C))
    lens = {}
    for lab, arr in ((lab_a, a), (lab_b, b), (lab_c, c)):
        for x, n in zip(lab, arr.shape):
            if lens.setdefault(x, n) != n:
                raise ValueError(f"length mismatch for {x!r}")
    labels = sorted(lens)
    acc = np.zeros(c.shape, dtype=np.float64)
    if alpha != 0.0:
        for values in itertools.product(*[range(lens[x]) for x in labels]):
            v = dict(zip(labels, values))
            acc[tuple(v[x] for x in lab_c)] += (a[tuple(v[x] for x in lab_a)] *
                                                 b[tuple(v[x] for x in lab_b)])
    return alpha * acc + (beta * c if beta != 0.0 else 0.0)


def flops(spec: str, lens: dict) -> int:
    """2 * n_I * n_J * n_P."""
    lab_c, lab_a, lab_b = _parse(spec)
    n = 1
    for x in set(lab_a) | set(lab_b) | set(lab_c):
        n *= lens[x]
    return 2 * n


def freivalds_dims(spec: str, A, B, C):
    """(n_I, n_J, n_P): extents of the I = C∩A, J = C∩B, P = A∩B label groups."""
    (a, b, c), _code, _keep = _args(spec, A, B, C)
    dims = (ctypes.c_int64 * 3)()
    err = _load().oracle_freivalds_dims(*a[1:], *b[1:], *c[1:], dims)
    if err:
        raise ValueError(f"oracle: {ERRORS.get(err, err)} for {spec!r}")
    return int(dims[0]), int(dims[1]), int(dims[2])


def freivalds(spec: str, A, B, C_new, C_old, x: np.ndarray, threads: Optional[int] = None):
    """Pin p8: the matrix-form products of oracle/contract.c's
    oracle_freivalds for one vector x over J (colexicographic over the J labels in C's order).
    Returns dict(u=B·x [n_P], v=A·u [n_I], wnew=C_new·x [n_I], wold=C_old·x [n_I] or None).
    C_old may be None (beta == 0: C_old is not read)."""
    (a, b, c), code, _keep = _args(spec, A, B, C_new)
    nI, nJ, nP = freivalds_dims(spec, A, B, C_new)
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.shape == (nJ,), (x.shape, nJ)
    sold, pold, keep2 = None, None, None
    if C_old is not None:
        p, lens, strides, code2 = _view(C_old)
        if code2 != code or lens != list(_view(C_new)[1]):
            raise ValueError("C_old must match C_new's dtype and shape")
        keep2 = _arr(strides)
        sold, pold = keep2, ctypes.c_void_p(p)
    u = np.zeros(max(nP, 1)); v = np.zeros(max(nI, 1))
    wn = np.zeros(max(nI, 1)); wo = np.zeros(max(nI, 1))
    DP = ctypes.POINTER(ctypes.c_double)
    err = _load().oracle_freivalds(code, *a, *b, *c, pold, sold,
                                   x.ctypes.data_as(DP), u.ctypes.data_as(DP),
                                   v.ctypes.data_as(DP), wn.ctypes.data_as(DP),
                                   wo.ctypes.data_as(DP), int(threads or 0))
    if err:
        raise ValueError(f"oracle: {ERRORS.get(err, err)} for {spec!r}")
    return dict(u=u[:nP], v=v[:nI], wnew=wn[:nI], wold=wo[:nI] if C_old is not None else None)


def freivalds_vectors(nJ: int, nvec: int = 3, seed: int = 0, lo: int = -1024, hi: int = 1024):
    """Seeded integer test vectors x in [lo, hi]^nJ, float64."""
    rs = np.random.RandomState(seed)
    return [rs.randint(lo, hi + 1, size=nJ).astype(np.float64) for _ in range(nvec)]


def frob(T) -> float:
    """Frobenius norm of a tensor's elements (the norm of its matrix form)."""
    try:
        import torch
        if isinstance(T, torch.Tensor):
            return float(torch.linalg.vector_norm(T.double() if T.dtype != torch.float64 else T))
    except ImportError:  # pragma: no cover
        pass
    return float(np.linalg.norm(np.asarray(T, dtype=np.float64).ravel()))


def freivalds_check(spec: str, A, B, C_new, C_old, alpha: float, beta: float, nvec: int = 3,
                    seed: int = 0, exact: bool = False, threads: Optional[int] = None):
    """Pin p8: for nvec seeded x, compare C_new·x with alpha·A·(B·x) + beta·C_old·x.
    exact=True (integer inputs, every partial sum exact): bitwise equality, returns 0.0 or the
    largest |difference|. Otherwise the normwise residual
      ||C_new·x − alpha·A·(B·x) − beta·C_old·x|| / (|alpha|·||A||_F·||B·x|| + |beta|·||C_old·x||)
    maximised over the vectors."""
    nI, nJ, nP = freivalds_dims(spec, A, B, C_new)
    worst = 0.0
    normA = None
    for x in freivalds_vectors(nJ, nvec, seed):
        r = freivalds(spec, A, B, C_new, C_old if beta != 0.0 else None, x, threads)
        rhs = alpha * r["v"]
        if beta != 0.0:
            rhs = rhs + beta * r["wold"]
        d = r["wnew"] - rhs
        if exact:
            worst = max(worst, float(np.abs(d).max()) if d.size else 0.0)
            continue
        if normA is None:
            normA = frob(A)
        den = abs(alpha) * normA * float(np.linalg.norm(r["u"]))
        if beta != 0.0:
            den += abs(beta) * float(np.linalg.norm(r["wold"]))
        num = float(np.linalg.norm(d))
        worst = max(worst, num / den if den > 0 else num)
    return worst
