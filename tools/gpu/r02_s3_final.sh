# Round-2 session-3 final records on the final build (after the cluster split-K coverage gate):
# ncu --set full of the cluster split-K path (fp64 512^3: 16 tiles, clusters of 8), the fp64 size
# sweep, and the f1 / f2 suites (no TTDT: its lines are in suite_r02s3_f2_final.jsonl)
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import torch, paper_1607_00291_b200 as tc
A = torch.randn(512, 512, device="cuda", dtype=torch.float64); B = torch.randn(512, 512, device="cuda", dtype=torch.float64)
C = torch.empty(512, 512, device="cuda", dtype=torch.float64)
for _ in range(3): tc.contract("mn-mk-kn", A, B, C)
torch.cuda.synchronize()
print("max err", (C - A @ B).abs().max().item())
PY
PYTHONPATH=$PWD timeout 300 python /tmp/one.py > gpurun_out/plain_csk512.log 2>&1 && \
PYTHONPATH=$PWD timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 2 -c 1 -o gpurun_out/prof_csk512 -f python /tmp/one.py > gpurun_out/ncu_csk512.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/plain_csk512.log
python tools/ncu_summary.py gpurun_out/prof_csk512.ncu-rep > gpurun_out/summary_csk512_f64.txt 2>&1
rm -f gpurun_out/prof_csk512.ncu-rep
SWEEP_DTYPE=f64 timeout 600 python tools/f32_size_sweep.py > gpurun_out/f64_size_sweep_final.jsonl 2> gpurun_out/f64_sweep.err; tail -3 gpurun_out/f64_size_sweep_final.jsonl | cut -c1-200
timeout 400 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_r02s3_f1_ck10.jsonl 2>/dev/null
timeout 500 python tools/suite.py --family f2 --no-ttdt > gpurun_out/suite_r02s3_f2_ck10.jsonl 2>/dev/null
python - <<'PY'
import json, statistics
for f in ("f2", "f1"):
    rows = [json.loads(l) for l in open(f"gpurun_out/suite_r02s3_{f}_ck10.jsonl")]
    v = [r["vs_gemm"] for r in rows if "vs_gemm" in r]
    print(f, len(rows), "median vs_gemm", statistics.median(v), "min", min(v))
PY
