"""paper_1607_00291_b200 -- transposition-free tensor contraction on B200 (sm_100a).

Thin ctypes binding over the C ABI in include/tc.h (libtc_b200.so). Argument marshalling only:
every step of the contraction (bundle classification, the section 7.3 heuristic, scatter and
block-scatter tables, staging, DMMA micro-kernel, epilogue) runs in the native library. There is
no CPU fallback: importing this package without the built library raises ImportError, and every
call that fails raises TCError.

    import paper_1607_00291_b200 as tc
    tc.contract("abcd-aebf-dfce", A, B, C, alpha=1.0, beta=0.0)   # torch CUDA tensors, C-A-B order

The index string lists the labels of C, A and B, in that order.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TC_B200_LIB") or os.path.join(_HERE, "libtc_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                      "(or __graft_entry__.build()) -- there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

TC_F64, TC_F32 = 0, 1
TC_MAX_RANK = 16
ERRORS = {0: "TC_OK", 1: "TC_ERR_ARG", 2: "TC_ERR_LABEL", 3: "TC_ERR_SHAPE", 4: "TC_ERR_ALIAS",
          5: "TC_ERR_UNSUPPORTED", 6: "TC_ERR_CUDA", 7: "TC_ERR_NOMEM"}
EXPORTS = ["tc_contract", "tc_contract_host", "tc_release_staging", "tc_plan_create", "tc_plan_execute",
           "tc_plan_destroy", "tc_plan_query", "tc_plan_dim", "tc_plan_scatter",
           "tc_plan_traversal_scatter",
           "tc_plan_block_scatter", "tc_error_string", "tc_last_error_detail", "tc_version"]

I64P = ctypes.POINTER(ctypes.c_int64)


class tc_tensor(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("lens", I64P), ("strides", I64P),
                ("labels", ctypes.c_char_p), ("data", ctypes.c_void_p)]


class tc_plan_info(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
                ("flops", ctypes.c_int64), ("swapped", ctypes.c_int32),
                ("ndims", ctypes.c_int32 * 3), ("a_vec_m", ctypes.c_int32),
                ("b_vec_k", ctypes.c_int32), ("idx64", ctypes.c_int32),
                ("variant", ctypes.c_int32)]


TP = ctypes.POINTER(tc_tensor)
_lib.tc_contract.argtypes = [ctypes.c_int, ctypes.c_double, TP, TP, ctypes.c_double, TP,
                             ctypes.c_void_p]
_lib.tc_contract_host.argtypes = _lib.tc_contract.argtypes
_lib.tc_plan_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, TP, TP, TP]
_lib.tc_plan_execute.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                 ctypes.c_void_p]
_lib.tc_plan_destroy.argtypes = [ctypes.c_void_p]
_lib.tc_plan_query.argtypes = [ctypes.c_void_p, ctypes.POINTER(tc_plan_info)]
_lib.tc_plan_dim.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, I64P, I64P, I64P,
                             ctypes.c_char_p, ctypes.c_int]
_lib.tc_plan_scatter.argtypes = [ctypes.c_void_p, ctypes.c_int, I64P, ctypes.c_int64, I64P]
_lib.tc_plan_traversal_scatter.argtypes = _lib.tc_plan_scatter.argtypes
_lib.tc_plan_block_scatter.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, I64P,
                                       ctypes.c_int64, I64P]
_lib.tc_error_string.argtypes = [ctypes.c_int]
_lib.tc_error_string.restype = ctypes.c_char_p
_lib.tc_last_error_detail.restype = ctypes.c_char_p
for _f in EXPORTS:
    if _f not in ("tc_error_string", "tc_last_error_detail"):
        getattr(_lib, _f).restype = ctypes.c_int


class TCError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        detail = _lib.tc_last_error_detail().decode(errors="replace")
        super().__init__(f"{ERRORS.get(code, code)}: {detail}")


def _check(rc: int) -> None:
    if rc != 0:
        raise TCError(rc)


class Desc:
    """A tc_tensor plus the ctypes arrays that keep its host fields alive."""

    def __init__(self, labels: str, lens: Sequence[int], strides: Sequence[int], data: int):
        if len(labels) != len(lens) or len(lens) != len(strides):
            raise ValueError(f"labels {labels!r} do not match rank {len(lens)}")
        n = max(len(lens), 1)
        self._lens = (ctypes.c_int64 * n)(*[int(x) for x in lens])
        self._strides = (ctypes.c_int64 * n)(*[int(x) for x in strides])
        self._labels = labels.encode()
        self.t = tc_tensor(len(lens), self._lens, self._strides, self._labels, ctypes.c_void_p(data))


def _dtype_code(dtype) -> int:
    import torch
    if dtype is torch.float64:
        return TC_F64
    if dtype is torch.float32:
        return TC_F32
    raise TypeError(f"unsupported dtype {dtype}")


def parse_spec(spec: str) -> Tuple[str, str, str]:
    """'C-A-B' index string -> (labels_C, labels_A, labels_B)."""
    parts = spec.split("-")
    if len(parts) != 3:
        raise ValueError(f"index string must be C-A-B, got {spec!r}")
    return parts[0], parts[1], parts[2]


_tls = __import__("threading").local()


def _desc(t, labels: str, role: int = 0) -> Desc:
    """Descriptor of a torch tensor; the lens/strides arrays are cached per thread by
    (operand role, labels, shape, strides) so repeated calls only refresh the data pointer."""
    cache = getattr(_tls, "descs", None)
    if cache is None:
        cache = _tls.descs = {}
    key = (role, labels, t.shape, t.stride())
    d = cache.get(key)
    if d is None:
        if len(cache) > 256:
            cache.clear()
        d = cache[key] = Desc(labels, list(t.shape), list(t.stride()), 0)
    d.t.data = t.data_ptr()
    return d


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    return stream.cuda_stream


def tc_contract(dtype: int, alpha: float, A: Desc, B: Desc, beta: float, C: Desc,
                stream: Optional[int]) -> None:
    """Direct binding of tc_contract (device pointers inside the descriptors)."""
    _check(_lib.tc_contract(dtype, float(alpha), ctypes.byref(A.t), ctypes.byref(B.t),
                            float(beta), ctypes.byref(C.t), stream))


def tc_contract_host(dtype: int, alpha: float, A: Desc, B: Desc, beta: float, C: Desc,
                     stream: Optional[int]) -> None:
    """Direct binding of tc_contract_host (host pointers; synchronous)."""
    _check(_lib.tc_contract_host(dtype, float(alpha), ctypes.byref(A.t), ctypes.byref(B.t),
                                 float(beta), ctypes.byref(C.t), stream))


_specs = {}
torch_C = None   # torch._C, bound on the first contract() call (the import stays torch-free)


def contract(spec: str, A, B, C, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """C := alpha * A.B + beta * C for torch CUDA tensors, asynchronously on `stream`
    (default: the current torch stream). Returns C.

    The descriptors of a (spec, dtype, shapes, strides) combination are built once per thread;
    a repeated call only refreshes the three data pointers before the C-ABI call (the library
    then finds its cached plan), which keeps the host cost of small contractions low."""
    fast = getattr(_tls, "fast", None)
    if fast is None:
        fast = _tls.fast = {}
    key = (spec, C.dtype, A.shape, A.stride(), B.shape, B.stride(), C.shape, C.stride())
    ent = fast.get(key)
    if ent is None:
        global torch_C
        if torch_C is None:
            import torch
            torch_C = torch._C
        labels = _specs.get(spec)
        if labels is None:
            labels = _specs[spec] = parse_spec(spec)
        lc, la, lb = labels
        dA = Desc(la, list(A.shape), list(A.stride()), 0)
        dB = Desc(lb, list(B.shape), list(B.stride()), 0)
        dC = Desc(lc, list(C.shape), list(C.stride()), 0)
        if len(fast) > 256:
            fast.clear()
        ent = fast[key] = (_dtype_code(C.dtype), dA.t, dB.t, dC.t, ctypes.byref(dA.t),
                           ctypes.byref(dB.t), ctypes.byref(dC.t), (dA, dB, dC))
    if not (A.is_cuda and B.is_cuda and C.is_cuda):
        raise ValueError("contract() takes CUDA tensors; use contract_host() for host memory")
    if A.dtype is not C.dtype or B.dtype is not C.dtype:
        raise TypeError(f"A, B, C must share one dtype (got {A.dtype}, {B.dtype}, {C.dtype})")
    dev = torch_C._cuda_getDevice()
    if A.get_device() != dev or B.get_device() != dev or C.get_device() != dev:
        raise ValueError(f"A, B, C must be on the current CUDA device (cuda:{dev}); got "
                         f"{A.device}, {B.device}, {C.device}")
    code, tA, tB, tC, pA, pB, pC, _ = ent
    tA.data = A.data_ptr()
    tB.data = B.data_ptr()
    tC.data = C.data_ptr()
    if stream is None:
        sp = torch_C._cuda_getCurrentRawStream(dev)
    else:
        sp = stream.cuda_stream
    rc = _lib.tc_contract(code, alpha, pA, pB, beta, pC, sp)
    if rc != 0:
        raise TCError(rc)
    return C


def contract_host(spec: str, A, B, C, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """End-to-end path on host tensors (pinned for full bandwidth): the library copies the
    operands to the current CUDA device, contracts, and copies C back (synchronous)."""
    lc, la, lb = parse_spec(spec)
    if A.dtype is not C.dtype or B.dtype is not C.dtype:
        raise TypeError(f"A, B, C must share one dtype (got {A.dtype}, {B.dtype}, {C.dtype})")
    if A.is_cuda or B.is_cuda or C.is_cuda:
        raise ValueError("contract_host() takes host tensors; use contract() for CUDA tensors")
    tc_contract_host(_dtype_code(C.dtype), alpha, _desc(A, la, 0), _desc(B, lb, 1), beta,
                     _desc(C, lc, 2), _stream_ptr(stream))
    return C


class Plan:
    """tc_plan_* wrapper. Creating a plan needs no GPU (structure only)."""

    def __init__(self, spec: str, dtype, shapes, strides):
        lc, la, lb = parse_spec(spec)
        (sa, sb, sc), (ta, tb, tcs) = shapes, strides
        self.spec = spec
        self._d = [Desc(la, sa, ta, 0), Desc(lb, sb, tb, 0), Desc(lc, sc, tcs, 0)]
        self._p = ctypes.c_void_p()
        code = dtype if isinstance(dtype, int) else _dtype_code(dtype)
        _check(_lib.tc_plan_create(ctypes.byref(self._p), code, ctypes.byref(self._d[0].t),
                                   ctypes.byref(self._d[1].t), ctypes.byref(self._d[2].t)))

    @classmethod
    def for_tensors(cls, spec: str, A, B, C) -> "Plan":
        return cls(spec, C.dtype, (list(A.shape), list(B.shape), list(C.shape)),
                   (list(A.stride()), list(B.stride()), list(C.stride())))

    def __del__(self):
        if getattr(self, "_p", None) and self._p.value and _lib is not None:
            _lib.tc_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def execute(self, A, B, C, alpha: float = 1.0, beta: float = 0.0, stream=None):
        if A.dtype is not C.dtype or B.dtype is not C.dtype:
            raise TypeError("A, B, C must share one dtype")
        _check(_lib.tc_plan_execute(self._p, float(alpha), A.data_ptr(), B.data_ptr(),
                                    float(beta), C.data_ptr(), _stream_ptr(stream)))
        return C

    def info(self) -> dict:
        i = tc_plan_info()
        _check(_lib.tc_plan_query(self._p, ctypes.byref(i)))
        return {"m": i.m, "n": i.n, "k": i.k, "flops": i.flops, "swapped": bool(i.swapped),
                "ndims": list(i.ndims), "a_vec_m": bool(i.a_vec_m), "b_vec_k": bool(i.b_vec_k),
                "idx64": bool(i.idx64), "variant": i.variant}

    def dims(self, which: int):
        """Folded dims of bundle which (0 I, 1 J, 2 P): [(labels, len, stride0, stride1)]."""
        out = []
        for idx in range(self.info()["ndims"][which]):
            ln, s0, s1 = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            buf = ctypes.create_string_buffer(TC_MAX_RANK + 2)
            _check(_lib.tc_plan_dim(self._p, which, idx, ctypes.byref(ln), ctypes.byref(s0),
                                    ctypes.byref(s1), buf, len(buf)))
            out.append((buf.value.decode(), ln.value, s0.value, s1.value))
        return out

    def scatter(self, which: int):
        n = ctypes.c_int64()
        _check(_lib.tc_plan_scatter(self._p, which, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_int64 * max(n.value, 1))()
        _check(_lib.tc_plan_scatter(self._p, which, arr, n.value, ctypes.byref(n)))
        return list(arr)[: n.value]

    def traversal_scatter(self, which: int):
        """The tables the kernel walks (GPU traversal order, reading R16)."""
        n = ctypes.c_int64()
        _check(_lib.tc_plan_traversal_scatter(self._p, which, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_int64 * max(n.value, 1))()
        _check(_lib.tc_plan_traversal_scatter(self._p, which, arr, n.value, ctypes.byref(n)))
        return list(arr)[: n.value]

    def block_scatter(self, which: int, b: int):
        n = ctypes.c_int64()
        _check(_lib.tc_plan_block_scatter(self._p, which, b, None, 0, ctypes.byref(n)))
        arr = (ctypes.c_int64 * max(n.value, 1))()
        _check(_lib.tc_plan_block_scatter(self._p, which, b, arr, n.value, ctypes.byref(n)))
        return list(arr)[: n.value]


SCATTER_NAMES = ["rscat_A", "cscat_A", "rscat_B", "cscat_B", "rscat_C", "cscat_C"]


def release_staging() -> None:
    """Free the device staging memory contract_host keeps between calls (tc_release_staging)."""
    _check(_lib.tc_release_staging())


def version() -> int:
    return _lib.tc_version()
