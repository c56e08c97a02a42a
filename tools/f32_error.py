"""Normwise relative error of the fp32 paths at cfg4's full fp32 sizes: the library's result
against torch.einsum of the same inputs widened to fp64 (on the GPU; measurement only, not a
parity test -- tests/test_gpu_parity.py holds those). One JSON line per case.

    TC_F32_UMMA=1 python tools/f32_error.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402


def main():
    for i in range(20):
        case = W.cfg4(i, torch.float32)
        A, B, C = W.make_tensors(case, "cuda")
        C0 = C.clone()
        tc.contract(case.spec, A, B, C, case.alpha, case.beta)
        la, lb, lc = case.lab_a, case.lab_b, case.lab_c
        ref = torch.einsum(f"{la},{lb}->{lc}", A.double(), B.double()) * case.alpha
        if case.beta != 0:
            ref += case.beta * C0.double()
        e = ((C.double() - ref).norm() / ref.norm()).item()
        emax = ((C.double() - ref).abs().max() / ref.abs().max()).item()
        print(json.dumps({"config": case.name, "umma": os.environ.get("TC_F32_UMMA", ""),
                          "normwise": e, "max_rel_to_max": emax}), flush=True)
        del A, B, C, C0, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
