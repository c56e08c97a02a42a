"""Table of vs_gemm across gpurun_out/v_<name>.jsonl files.  python tools/compare_many.py a b c"""
import json
import sys

names = sys.argv[1:]
R = []
for n in names:
    d = {}
    for line in open(f"gpurun_out/v_{n}.jsonl"):
        try:
            x = json.loads(line)
            d[x["config"]] = x
        except ValueError:
            pass
    R.append(d)
print(f"{'config':34s} " + " ".join(f"{n:>9s}" for n in names))
for k in R[0]:
    print(f"{k[:34]:34s} " + " ".join(f"{r.get(k, {}).get('vs_gemm', 0):9.3f}" for r in R))
