"""Quick correctness / speed check of one fp32 tcgen05 form (TC_UMMA_FORM) on GEMM layouts and a
few cfg4 fp32 cases, against fp64 torch on the GPU. Measurement helper, not a parity test."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402


def err(C, ref):
    return ((C.double() - ref).norm() / ref.norm()).item()


for (m, n, k) in [(256, 128, 64), (300, 200, 100), (1024, 1024, 1024), (4096, 4096, 4096)]:
    A = torch.randn(m, k, device="cuda"); B = torch.randn(k, n, device="cuda")
    C = torch.full((m, n), float("nan"), device="cuda")
    tc.contract("mn-mk-kn", A, B, C)
    torch.cuda.synchronize()
    e = err(C, A.double() @ B.double())
    t0 = time.perf_counter()
    for _ in range(5):
        tc.contract("mn-mk-kn", A, B, C)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(json.dumps({"mnk": [m, n, k], "err": e, "ms": round(ms, 4),
                      "tflops": round(2 * m * n * k / ms / 1e9, 1)}), flush=True)
for i in (0, 8, 11, 19):
    case = W.cfg4(i, torch.float32)
    A, B, C = W.make_tensors(case, "cuda")
    tc.contract(case.spec, A, B, C, case.alpha, case.beta)
    ref = torch.einsum(f"{case.lab_a},{case.lab_b}->{case.lab_c}", A.double(), B.double())
    print(json.dumps({"case": case.name, "err": err(C, ref)}), flush=True)
