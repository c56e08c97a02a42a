import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1607_00291_b200 as tc
n = int(sys.argv[1])
A = torch.randn(n, n, device="cuda"); B = torch.randn(n, n, device="cuda"); C = torch.empty(n, n, device="cuda")
tc.contract("mn-mk-kn", A, B, C); torch.cuda.synchronize()
print("--- timed", flush=True)
tc.contract("mn-mk-kn", A, B, C); torch.cuda.synchronize()
