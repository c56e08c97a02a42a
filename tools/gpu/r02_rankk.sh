# rank-k kernel v2 (persistent, cp.async offset/value rings) vs v1 (TC_RANKK_V=1): parity, then f1
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "rankk or f1" > gpurun_out/rk_parity.log 2>&1; tail -2 gpurun_out/rk_parity.log
python - <<'PY'
import torch, time
C = torch.empty(16000 * 16000, dtype=torch.float64, device="cuda")
for _ in range(3): C.fill_(1.0)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): C.fill_(1.0)
e1.record(); torch.cuda.synchronize()
print("torch fill_ write bandwidth GB/s:", round(C.numel() * 8 * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1))
PY
timeout 600 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_rk2.jsonl 2>/dev/null
TC_RANKK_V=1 timeout 600 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_rk1.jsonl 2>/dev/null
for O in 8 16 64 128; do TC_RANKK_OCC2=$O timeout 600 python tools/suite.py --family f1 --only f1_k5 --no-ttdt | sed "s/^/occ$O /"; done
python - <<'PY'
import json
a = [json.loads(l) for l in open("gpurun_out/suite_rk1.jsonl")]
b = [json.loads(l) for l in open("gpurun_out/suite_rk2.jsonl")]
for x, y in zip(a, b):
    print(f"{x['config'][:30]:30s} v1 {x['ms']:8.4f} ms {x['hbm_gbs']:7.0f} GB/s {x['vs_gemm']:6.3f}   v2 {y['ms']:8.4f} ms {y['hbm_gbs']:7.0f} GB/s {y['vs_gemm']:6.3f}")
PY
