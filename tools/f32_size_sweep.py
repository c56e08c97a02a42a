"""Contraction time over square-ish GEMM-layout sizes for the current fp32 path (TC_F32_UMMA=0/1)
or fp64 (SWEEP_DTYPE=f64), next to cuBLAS of equal M, N, K; CUDA graphs of 20 calls, one JSON
line per size.

    TC_F32_UMMA=0 python tools/f32_size_sweep.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402


def graph_ms(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * n)


def main():
    sizes = [(256, 256, 256), (512, 512, 512), (768, 768, 768), (1024, 1024, 1024),
             (1536, 1536, 1536), (2048, 2048, 2048), (4096, 4096, 4096),
             (4096, 4096, 64), (8192, 8192, 256), (256, 256, 65536)]
    if os.environ.get("SWEEP_SIZES"):   # e.g. "512x512x512,1024x1024x1024"
        sizes = [tuple(int(v) for v in t.split("x")) for t in os.environ["SWEEP_SIZES"].split(",")]
    dt = torch.float64 if os.environ.get("SWEEP_DTYPE") == "f64" else torch.float32
    for m, n, k in sizes:
        A = torch.randn(m, k, device="cuda", dtype=dt)
        B = torch.randn(k, n, device="cuda", dtype=dt)
        C = torch.empty(m, n, device="cuda", dtype=dt)
        t = graph_ms(lambda: tc.contract("mn-mk-kn", A, B, C))
        tg = graph_ms(lambda: torch.mm(A, B, out=C))
        fl = 2.0 * m * n * k
        print(json.dumps({"mnk": [m, n, k], "dtype": str(dt).split(".")[-1],
                          "umma": os.environ.get("TC_F32_UMMA", "1"),
                          "ms": round(t, 4), "tflops": round(fl / t / 1e9, 2),
                          "gemm_ms": round(tg, 4), "vs_gemm": round(tg / t, 3)}), flush=True)


if __name__ == "__main__":
    main()
