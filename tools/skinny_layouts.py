"""Skinny-kernel component timings (TC_SKINNY_DBG: 1 no MMA, 2 no X loads, 4 no C stores) on the
fig:bench f2_00 layout (sub-divided rows: 64-byte runs of X and C) next to the plain column-major
GEMM layout of the same M, N, K (X and C contiguous along M). Measurement only.

    python tools/skinny_layouts.py > gpurun_out/skinny_layouts.jsonl
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402
from suite import timeit  # noqa: E402

cases = [W.fig_bench(0),
         W.Case("plain_mn-mk-kn", "mn", "mk", "kn", {"m": 2 ** 20, "n": 32, "k": 32},
                dist="uniform", alpha=1.0, beta=0.0, c_init="nan", seed=5)]
for case in cases:
    A, B, C = W.make_tensors(case, "cuda")
    for dbg in ["0", "1", "2", "4", "3", "5", "6"]:
        os.environ["TC_SKINNY_DBG"] = dbg
        ms = timeit(lambda: tc.contract(case.spec, A, B, C, case.alpha, case.beta), 20)
        print(json.dumps({"case": case.name, "dbg": int(dbg), "us": round(ms * 1e3, 1),
                          "ws": os.environ.get("TC_SKINNY_WS", "")}), flush=True)
    os.environ["TC_SKINNY_DBG"] = "0"
