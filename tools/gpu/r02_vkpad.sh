# fp32: 16-byte K-chunk pad under the K-vector gathers (mode 2), A/B against -DTC_UMMA_VKPAD16=0
mkdir -p gpurun_out
TC_LIB_OUT=/tmp/tc_vk64.so TC_NVCC_EXTRA="-DTC_UMMA_VKPAD16=0" python paper_1607_00291_b200/_build.py > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard" 2>&1 | tail -1
for r in 1 2; do
  timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/vk16_$r.jsonl 2>/dev/null
  TC_B200_LIB=/tmp/tc_vk64.so timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/vk64_$r.jsonl 2>/dev/null
done
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
a = [load(f"gpurun_out/vk16_{r}.jsonl") for r in (1, 2)]
b = [load(f"gpurun_out/vk64_{r}.jsonl") for r in (1, 2)]
for k in a[0]:
    print(f"{k[:34]:34s} pad16 {a[0][k]['gflops']/1e3:6.1f} {a[1][k]['gflops']/1e3:6.1f}  pad64 {b[0][k]['gflops']/1e3:6.1f} {b[1][k]['gflops']/1e3:6.1f}")
print("median pad16", round(st.median(v["gflops"] for v in a[0].values())/1e3, 1), "pad64", round(st.median(v["gflops"] for v in b[0].values())/1e3, 1))
PY
