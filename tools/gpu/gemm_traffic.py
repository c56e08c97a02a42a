"""cuBLAS DGEMM of cfg5's M x N x K, for its DRAM traffic under ncu (comparison for the
contraction kernel's traffic, profiles/r01/traffic_*.csv)."""
import torch
m, n, k = 55296, 27648, 27648
a = torch.randn(m, k, dtype=torch.float64, device="cuda")
b = torch.randn(k, n, dtype=torch.float64, device="cuda")
c = torch.empty(m, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.mm(a, b, out=c)
torch.cuda.synchronize()
print("ok")
