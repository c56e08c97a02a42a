"""Side-by-side of two tools/suite.py outputs: GFLOP/s and ratio to the same-size GEMM.
    python tools/compare_suites.py new.jsonl old.jsonl"""
import json
import sys


def load(p):
    out = {}
    for line in open(p):
        try:
            d = json.loads(line)
        except ValueError:
            continue
        out[d["config"]] = d
    return out


a, b = load(sys.argv[1]), load(sys.argv[2])
for k, d in a.items():
    o = b.get(k, {})
    print(f"{k[:36]:36s} {str(d['mnk']):22s} {d['gflops']:9.0f} ({d['vs_gemm']:.3f})   "
          f"{o.get('gflops', 0):9.0f} ({o.get('vs_gemm', 0):.3f})  gemm {d['gemm_gflops']:8.0f}")
