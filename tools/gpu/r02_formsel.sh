mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ablation.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard or forced or epoch or fresh or concurrent" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" 2>&1 | tail -1
for r in 1 2; do timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/formsel_$r.jsonl 2>/dev/null; done
SWEEP_DTYPE=f32 timeout 600 python tools/f32_size_sweep.py > gpurun_out/formsel_sweep.jsonl 2>/dev/null; cat gpurun_out/formsel_sweep.jsonl | cut -c1-160
python - <<'PY'
import json, math, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
for r in (1, 2):
    d = load(f"gpurun_out/formsel_{r}.jsonl"); v = [x["gflops"] for x in d.values()]
    print(r, "median", round(st.median(v)/1e3, 1), "geomean", round(math.exp(sum(math.log(x) for x in v)/len(v))/1e3, 1), "min", round(min(v)/1e3,1), "vs_sgemm median", st.median(x["vs_gemm"] for x in d.values()))
PY
