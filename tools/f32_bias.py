"""Normwise error of the fp32 path on one-signed data (uniform [0, 1)), where rounding biases
add up instead of cancelling: C = A B for m = n = 512 and growing K, against fp64 on the GPU.

    TC_F32_UMMA=0|1 [TC_B200_LIB=variant.so] python tools/f32_bias.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(7)
    for k in (64, 1024, 8192, 65536):
        A = torch.rand(512, k, device="cuda", generator=g)
        B = torch.rand(k, 512, device="cuda", generator=g)
        C = torch.empty(512, 512, device="cuda")
        tc.contract("mn-mk-kn", A, B, C)
        ref = A.double() @ B.double()
        e = ((C.double() - ref).norm() / ref.norm()).item()
        bias = ((C.double() - ref).sum() / ref.sum()).item()
        print(json.dumps({"k": k, "umma": os.environ.get("TC_F32_UMMA", "1"),
                          "lib": os.path.basename(os.environ.get("TC_B200_LIB", "default")),
                          "normwise": e, "mean_rel_bias": bias}), flush=True)


if __name__ == "__main__":
    main()
