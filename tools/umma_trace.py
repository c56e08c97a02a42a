"""One fp32 contraction (mn-mk-kn, sizes from argv) through a library built with -DTC_UMMA_TRACE;
prints the per-work-item timeline (relative us) of the fp32 tcgen05 kernel's epilogue."""
import os
import re
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1607_00291_b200 as tc
    m, n, k = (int(v) for v in sys.argv[2:5])
    A = torch.randn(m, k, device="cuda"); B = torch.randn(k, n, device="cuda")
    C = torch.empty(m, n, device="cuda")
    tc.contract("mn-mk-kn", A, B, C); torch.cuda.synchronize()
    print("--- second call", flush=True)
    tc.contract("mn-mk-kn", A, B, C); torch.cuda.synchronize()
    sys.exit(0)
out = subprocess.run([sys.executable, __file__, "--child", *sys.argv[1:4]], capture_output=True,
                     text=True).stdout
out = out.split("--- second call")[-1]
rows = [list(map(int, re.findall(r"\s(-?\d+)", l))) for l in out.splitlines() if l.startswith("TR")]
t0 = min(r[5] for r in rows)
for r in sorted(rows, key=lambda r: (r[0], r[5])):
    cta, tile, kb, ke, piece, st, w0, w1, en = r
    f = lambda t: (t - t0) / 1e3 if t else -1
    print(f"cta {cta:3d} tile {tile:3d} k[{kb:3d},{ke:3d}) piece {piece}  start {f(st):7.2f}"
          f"  wait {f(w0):7.2f}->{f(w1):7.2f}  end {f(en):7.2f}")
