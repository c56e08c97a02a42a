mkdir -p gpurun_out
TC_LIB_OUT=/tmp/tc_vk16.so TC_NVCC_EXTRA="-DTC_UMMA_VKPAD16=1" python paper_1607_00291_b200/_build.py > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; exit 1; }
TC_B200_LIB=/tmp/tc_vk16.so TC_UMMA_KV=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32_vector or f32_loader" 2>&1 | tail -1
TC_B200_LIB=/tmp/tc_vk16.so TC_UMMA_KV=1 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/kv16_on.jsonl 2>/dev/null
timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/kv16_off.jsonl 2>/dev/null
TC_B200_LIB=/tmp/tc_vk16.so TC_UMMA_KV=1 SWEEP_DTYPE=f32 timeout 600 python tools/f32_size_sweep.py 2>/dev/null | cut -c1-100 | tail -4
python - <<'PY'
import json, math, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
on, off = load("gpurun_out/kv16_on.jsonl"), load("gpurun_out/kv16_off.jsonl")
for k in on: print(f"{k[:34]:34s} kv-pad16 {on[k]['gflops']/1e3:6.1f}  default {off[k]['gflops']/1e3:6.1f}")
for n, d in (("kv-pad16", on), ("default", off)):
    v = [x["gflops"] for x in d.values()]
    print(n, "median", round(st.median(v)/1e3, 1), "geomean", round(math.exp(sum(math.log(x) for x in v)/len(v))/1e3, 1))
PY
