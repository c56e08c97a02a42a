# fp64 medium sizes: sweep + ncu of 512^3 (the DMMA tile kernel's few-tile regime)
mkdir -p gpurun_out
SWEEP_DTYPE=f64 SWEEP_SIZES=512x512x512 timeout 300 python tools/f32_size_sweep.py
cat > /tmp/one.py <<'PY'
import torch, paper_1607_00291_b200 as tc
A = torch.randn(512, 512, device="cuda", dtype=torch.float64); B = torch.randn(512, 512, device="cuda", dtype=torch.float64)
C = torch.empty(512, 512, device="cuda", dtype=torch.float64)
for _ in range(3): tc.contract("mn-mk-kn", A, B, C)
torch.cuda.synchronize()
PY
PYTHONPATH=$PWD timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 2 -c 1 -o gpurun_out/f64_512 -f python /tmp/one.py > gpurun_out/ncu_512.log 2>&1; echo ncu $?
