"""End-to-end host path (tc_contract_host, pinned host buffers, H2D + D2H inside the timed region)
on cfg5 for several chunk counts (TC_HOST_CHUNKS), CUDA events around synchronous calls."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402

case = W.cfg5()
Ad, Bd, _ = W.make_tensors(case, "cuda")
hA = W.colmajor_view(torch.empty(Ad.numel(), dtype=torch.float64, pin_memory=True), list(Ad.shape))
hB = W.colmajor_view(torch.empty(Bd.numel(), dtype=torch.float64, pin_memory=True), list(Bd.shape))
hA.copy_(Ad); hB.copy_(Bd)
del Ad, Bd
torch.cuda.empty_cache()
cs = case.shape(case.lab_c)
hC = W.colmajor_view(torch.empty(int(torch.tensor(cs).prod()), dtype=torch.float64, pin_memory=True), cs)
for n in [int(x) for x in sys.argv[1:]] or [8, 12, 16, 24]:
    os.environ["TC_HOST_CHUNKS"] = str(n)
    tc.contract_host(case.spec, hA, hB, hC)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        tc.contract_host(case.spec, hA, hB, hC)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(json.dumps({"chunks": n, "ms": round(ms, 1), "e2e_gflops": round(case.flops() / ms / 1e6, 1)}), flush=True)
