"""cuBLAS DGEMM ceiling on this box: the same-size GEMM of each
BASELINE.json config, timed with CUDA events. Not part of the product path."""
import json
import sys

import torch


def bench(m, n, k, reps=5, beta=0.0):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.addmm(c, a, b, beta=beta, alpha=1.0, out=c) if beta else torch.mm(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if beta:
            torch.addmm(c, a, b, beta=beta, alpha=1.0, out=c)
        else:
            torch.mm(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    torch.cuda.empty_cache()
    return best


if __name__ == "__main__":
    shapes = [(2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (16384, 1024, 16384),
              (13824, 13824, 27648)]
    if len(sys.argv) > 1 and sys.argv[1] == "--big":
        shapes.append((55296, 27648, 27648))
    for (m, n, k) in shapes:
        ms = bench(m, n, k, reps=3 if m * n * k > 1e12 else 10)
        print(json.dumps({"kind": "cublas_dgemm", "m": m, "n": n, "k": k, "ms": round(ms, 4),
                          "tflops": round(2 * m * n * k / ms / 1e9, 2)}), flush=True)
