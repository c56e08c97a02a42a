"""Top stalled SASS instructions of an `ncu --page source --csv` export, with context lines,
plus samples per opcode.   python tools/ncu_source_top.py gpurun_out/source_x.csv [N] [CTX]"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 12
CTX = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si] or 0) for r in body)
ops = Counter()
for r in body:
    op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    ops[op.split(".")[0]] += int(r[si] or 0)
print(f"total samples {tot}")
print("samples per opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in ops.most_common(14)))
order = sorted(range(len(body)), key=lambda i: -int(body[i][si] or 0))[:N]
for i in sorted(order):
    r = body[i]
    reasons = sorted(((int(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:3]
    print(f"--- {100*int(r[si])/tot:.2f}%  " + ", ".join(f"{n} {v}" for v, n in reasons if v))
    for j in range(max(0, i - CTX), min(len(body), i + 2)):
        mark = ">>" if j == i else "  "
        print(f"{mark} {body[j][0][-5:]} {int(body[j][si] or 0):6d} ex={body[j][ei]:>8s} {body[j][1].strip()[:90]}")
