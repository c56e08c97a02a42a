cat > /tmp/one.py <<'PY'
import os, torch, paper_1607_00291_b200 as tc
for n in (256, 512, 768, 1024):
    A = torch.randn(n, n, device="cuda", dtype=torch.float64); B = torch.randn(n, n, device="cuda", dtype=torch.float64)
    C = torch.empty(n, n, device="cuda", dtype=torch.float64)
    for S in ("8", "16"):
        os.environ["TC_CSK_MAX"] = S
        tc.contract("mn-mk-kn", A, B, C); torch.cuda.synchronize()
PY
TC_CSK_DEBUG=1 PYTHONPATH=$PWD python /tmp/one.py
PYTHONPATH=$PWD timeout 300 ncu --set full --clock-control none -k regex:tc_dmma -s 3 -c 1 -o gpurun_out/csk_512 -f python - <<'PY' > /dev/null 2>&1
import torch, paper_1607_00291_b200 as tc
A = torch.randn(512, 512, device="cuda", dtype=torch.float64); B = torch.randn(512, 512, device="cuda", dtype=torch.float64)
C = torch.empty(512, 512, device="cuda", dtype=torch.float64)
for _ in range(5): tc.contract("mn-mk-kn", A, B, C)
torch.cuda.synchronize()
PY
echo ncu $?
