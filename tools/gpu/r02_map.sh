# fp32 tcgen05 kernel: one-line-per-instruction element gathers (modes 7/8) vs TC_UMMA_MAP=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ablation.py tests/test_gpu_robustness.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard or forced or epoch or fresh" > gpurun_out/map_parity.log 2>&1; tail -1 gpurun_out/map_parity.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" > gpurun_out/map_full.log 2>&1; tail -1 gpurun_out/map_full.log
for r in 1 2; do
  timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/map_on_$r.jsonl 2>/dev/null
  TC_UMMA_MAP=0 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/map_off_$r.jsonl 2>/dev/null
done
TC_UMMA_FORM=128 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/map_on_f128.jsonl 2>/dev/null
TC_UMMA_FORM=256 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/map_on_f256.jsonl 2>/dev/null
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
on = [load(f"gpurun_out/map_on_{r}.jsonl") for r in (1, 2)]
off = [load(f"gpurun_out/map_off_{r}.jsonl") for r in (1, 2)]
f128, f256 = load("gpurun_out/map_on_f128.jsonl"), load("gpurun_out/map_on_f256.jsonl")
print("config                              on1     on2    off1    off2   f128   f256  (TF/s)")
for k in on[0]:
    print(f"{k[:34]:34s} {on[0][k]['gflops']/1e3:6.1f} {on[1][k]['gflops']/1e3:6.1f} {off[0][k]['gflops']/1e3:6.1f} {off[1][k]['gflops']/1e3:6.1f} {f128[k]['gflops']/1e3:6.1f} {f256[k]['gflops']/1e3:6.1f}")
for n, d in (("on", on[0]), ("off", off[0]), ("f128", f128), ("f256", f256)):
    print(n, "median", round(st.median(v["gflops"] for v in d.values()) / 1e3, 1))
PY
