# fp64 DMMA kernel: edge tiles multiply only the m16 / n8 blocks that hold data
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_ablation.py -m gpu -q -x -p no:cacheprovider -k "not f32" > gpurun_out/edge_parity.log 2>&1; tail -1 gpurun_out/edge_parity.log
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f64 or f2 or cfg2 or cfg3" > gpurun_out/edge_full.log 2>&1; tail -1 gpurun_out/edge_full.log
timeout 900 python tools/suite.py --family f2 --no-ttdt > gpurun_out/suite_edge_f2.jsonl 2>/dev/null
timeout 900 python tools/suite.py --no-ttdt --match "cfg4_.._f64" > gpurun_out/suite_edge_cfg4.jsonl 2>/dev/null
python - <<'PY'
import json
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
old = load("profiles/r02/suite_r02_f2.jsonl"); old.update(load("profiles/r02/suite_r02_baseline.jsonl"))
for f in ("gpurun_out/suite_edge_f2.jsonl", "gpurun_out/suite_edge_cfg4.jsonl"):
    for k, d in load(f).items():
        o = old.get(k, {})
        print(f"{k[:34]:34s} old {o.get('vs_gemm',0):6.3f} new {d['vs_gemm']:6.3f}  ({d['gflops']/1e3:6.2f} TF/s)")
PY
SWEEP_DTYPE=f64 timeout 600 python tools/f32_size_sweep.py 2>/dev/null | tail -12
