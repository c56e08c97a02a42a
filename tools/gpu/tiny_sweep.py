"""Tile kernel (TC_TINY=0) vs tiny kernel (limits raised) on small GEMM-like contractions:
CUDA-event time per call in a CUDA graph of 20 calls (kernel latency, no host overhead)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00291_b200 as tc  # noqa: E402


def graph_time(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 100


for dt in (torch.float64, torch.float32):
    for m, n, k in [(64, 64, 64), (128, 128, 128), (128, 128, 512), (256, 256, 256),
                    (256, 256, 1024), (512, 512, 512), (256, 256, 64), (512, 512, 64)]:
        A = torch.randn(m, k, dtype=dt, device="cuda")
        B = torch.randn(k, n, dtype=dt, device="cuda")
        C = torch.empty(m, n, dtype=dt, device="cuda")
        out = {"dtype": str(dt).split(".")[-1], "mnk": [m, n, k]}
        for name, env in (("tile", "0"), ("tiny", "1")):
            os.environ["TC_TINY"] = env
            out[name + "_us"] = round(graph_time(lambda: tc.contract("mn-mk-kn", A, B, C)), 2)
        out["cublas_us"] = round(graph_time(lambda: torch.mm(A, B, out=C)), 2)
        print(json.dumps(out), flush=True)
