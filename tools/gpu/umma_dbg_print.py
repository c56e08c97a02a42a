import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_1607_00291_b200 as tc
os.environ["TC_TINY"] = "0"; os.environ["TC_SKINNY"] = "0"; os.environ["TC_F32_UMMA"] = "1"
for spec in ["mn-mk-nk", "mn-km-kn"]:
    lc, la, lb = spec.split("-")
    d = {"m": 128, "n": 128, "k": 32}
    A = torch.arange(128 * 32, device="cuda", dtype=torch.float32).reshape([d[x] for x in la]) / 4096
    B = torch.ones([d[x] for x in lb], device="cuda")
    C = torch.full([d[x] for x in lc], float("nan"), device="cuda")
    tc.contract(spec, A, B, C)
    torch.cuda.synchronize()
    ref = torch.einsum(f"{la},{lb}->{lc}", A, B)
    print(spec, "C[0,0]", C[0, 0].item(), "ref", ref[0, 0].item(), "C[5,7]", C[5, 7].item(), ref[5, 7].item(), flush=True)
