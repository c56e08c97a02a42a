# fp32 N = 256 default: K vectors (TC_UMMA_KV=1) vs pairs / one-line K gathers; parity of the default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ablation.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard or forced or epoch or fresh or concurrent" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" 2>&1 | tail -1
TC_UMMA_KV=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32_vector or f32_loader" 2>&1 | tail -1
for r in 1 2; do
  timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/kv_off_$r.jsonl 2>/dev/null
  TC_UMMA_KV=1 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/kv_on_$r.jsonl 2>/dev/null
done
SWEEP_DTYPE=f32 timeout 600 python tools/f32_size_sweep.py > gpurun_out/kv_sweep_off.jsonl 2>/dev/null
SWEEP_DTYPE=f32 TC_UMMA_KV=1 timeout 600 python tools/f32_size_sweep.py > gpurun_out/kv_sweep_on.jsonl 2>/dev/null
python - <<'PY'
import json, math, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
on = [load(f"gpurun_out/kv_on_{r}.jsonl") for r in (1, 2)]
off = [load(f"gpurun_out/kv_off_{r}.jsonl") for r in (1, 2)]
for k in on[0]:
    print(f"{k[:34]:34s} kv {on[0][k]['gflops']/1e3:6.1f} {on[1][k]['gflops']/1e3:6.1f}  no-kv {off[0][k]['gflops']/1e3:6.1f} {off[1][k]['gflops']/1e3:6.1f}")
for n, d in (("kv", on[0]), ("no-kv", off[0])):
    v = [x["gflops"] for x in d.values()]
    print(n, "median", round(st.median(v)/1e3, 1), "geomean", round(math.exp(sum(math.log(x) for x in v)/len(v))/1e3, 1))
a = [json.loads(l) for l in open("gpurun_out/kv_sweep_off.jsonl")]; b = [json.loads(l) for l in open("gpurun_out/kv_sweep_on.jsonl")]
for x, y in zip(a, b): print(x["mnk"], "no-kv", x["tflops"], "kv", y["tflops"], "sgemm ratio", x["vs_gemm"])
PY
