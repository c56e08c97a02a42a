# fp32 N = 256 form: B along N by 16-byte vectors / 8-byte pairs into a [k][n] staging (modes 10/11)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ablation.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard or forced" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" 2>&1 | tail -1
for r in 1 2; do
  timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/bn_on_$r.jsonl 2>/dev/null
  TC_UMMA_BN=0 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/bn_off_$r.jsonl 2>/dev/null
done
python - <<'PY'
import json, math, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
on = [load(f"gpurun_out/bn_on_{r}.jsonl") for r in (1, 2)]
off = [load(f"gpurun_out/bn_off_{r}.jsonl") for r in (1, 2)]
for k in on[0]:
    print(f"{k[:34]:34s} on {on[0][k]['gflops']/1e3:6.1f} {on[1][k]['gflops']/1e3:6.1f}  off {off[0][k]['gflops']/1e3:6.1f} {off[1][k]['gflops']/1e3:6.1f}")
for n, d in (("on", on[0]), ("off", off[0])):
    v = [x["gflops"] for x in d.values()]
    print(n, "median", round(st.median(v)/1e3, 1), "geomean", round(math.exp(sum(math.log(x) for x in v)/len(v))/1e3, 1))
PY
