"""cfg1 (64^3) call latency: CUDA-event time per call for back-to-back tc.contract / Plan.execute
calls, host time per call, and the same calls captured in a CUDA graph (kernel-only latency)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402

case = W.cfg1()
A, B, C = W.make_tensors(case, "cuda")
s = torch.cuda.current_stream()
plan = tc.Plan.for_tensors(case.spec, A, B, C)
out = {}
def skinny_call():
    os.environ["TC_SKINNY"] = "1"
    tc.contract(case.spec, A, B, C, 1.0, 0.0)
    os.environ["TC_SKINNY"] = "0"


for name, fn in (("contract", lambda: tc.contract(case.spec, A, B, C, 1.0, 0.0)),
                 ("contract_skinny", skinny_call),
                 ("plan_execute", lambda: plan.execute(A, B, C, 1.0, 0.0)),
                 ("torch_mm_64", None)):
    if fn is None:
        a = torch.randn(64, 64, dtype=torch.float64, device="cuda")
        b = torch.randn(64, 64, dtype=torch.float64, device="cuda")
        c = torch.empty(64, 64, dtype=torch.float64, device="cuda")
        fn = lambda: torch.mm(a, b, out=c)  # noqa: E731
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out[name] = {"event_us": round(1e3 * e0.elapsed_time(e1) / n, 2),
                 "host_us": round(1e6 * (t1 - t0) / n, 2)}
# graph capture of the contraction: device time per replayed call
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(s)
with torch.cuda.stream(side):
    for _ in range(3):
        tc.contract(case.spec, A, B, C, 1.0, 0.0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            tc.contract(case.spec, A, B, C, 1.0, 0.0)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    g.replay()
e1.record(s)
torch.cuda.synchronize()
out["graph_per_call_us"] = round(1e3 * e0.elapsed_time(e1) / 200, 2)
print(json.dumps(out))
