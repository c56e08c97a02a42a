"""Run one contraction a few times (for ncu DRAM / L2 metrics): `cfg5` or `gemm5` (a dense
column-major GEMM with cfg5's M, N, K through the same kernel).
    python tools/gpu/traffic_probe.py cfg5|gemm5 [reps]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if which == "cfg5":
    case = W.cfg5()
else:
    case = W.Case("gemm5", "mn", "mk", "kn", {"m": 55296, "n": 27648, "k": 27648},
                  dist="normal", alpha=1.0, beta=0.0, c_init="zero", seed=1)
A, B, C = W.make_tensors(case, "cuda")
for _ in range(reps):
    tc.contract(case.spec, A, B, C, case.alpha, case.beta)
torch.cuda.synchronize()
print("ok", which)
