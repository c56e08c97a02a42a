"""Debug the tcgen05 3xTF32 fp32 path on plain GEMM layouts."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00291_b200 as tc  # noqa: E402

os.environ["TC_TINY"] = "0"
os.environ["TC_SKINNY"] = "0"
torch.manual_seed(0)
for spec in ["mn-mk-kn", "mn-km-nk", "mn-mk-nk", "mn-km-kn"]:
    for (m, n, k) in [(128, 128, 32), (256, 384, 100), (1000, 700, 513)]:
        lc, la, lb = spec.split("-")
        dims = {"m": m, "n": n, "k": k}
        A = torch.rand([dims[x] for x in la], device="cuda") * 2 - 1
        B = torch.rand([dims[x] for x in lb], device="cuda") * 2 - 1
        A = A.t().contiguous().t() if False else A
        ref = torch.einsum(f"{la},{lb}->{lc}", A.double(), B.double())
        out = {}
        for mode in ("0", "1"):
            os.environ["TC_F32_UMMA"] = mode
            C = torch.full([dims[x] for x in lc], float("nan"), device="cuda")
            tc.contract(spec, A, B, C)
            torch.cuda.synchronize()
            err = ((C.double() - ref).norm() / ref.norm()).item()
            out[mode] = (err, C[0, 0].item(), C[-1, -1].item())
        print(spec, (m, n, k), "ref", round(ref[0, 0].item(), 5), round(ref[-1, -1].item(), 5),
              "ffma", out["0"], "umma", out["1"], flush=True)
