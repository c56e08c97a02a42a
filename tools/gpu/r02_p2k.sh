# fp32 K-pair gathers 2 rows x 16 pairs (this build) vs the previous suite (profiles/r02/suite_f32_lines.jsonl)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" 2>&1 | tail -1
for r in 1 2; do timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/p2k_$r.jsonl 2>/dev/null; done
TC_UMMA_PAIRS=0 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/p2k_off.jsonl 2>/dev/null
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
old = load("/root/repo/profiles/r02/suite_f32_p2k_prev.jsonl")
n1, n2, off = load("gpurun_out/p2k_1.jsonl"), load("gpurun_out/p2k_2.jsonl"), load("gpurun_out/p2k_off.jsonl")
for k in old:
    print(f"{k[:34]:34s} prev {old[k]['gflops']/1e3:6.1f}  new {n1[k]['gflops']/1e3:6.1f} {n2[k]['gflops']/1e3:6.1f}  pairs-off {off[k]['gflops']/1e3:6.1f}")
for n, d in (("prev", old), ("new", n1), ("pairs-off", off)): print(n, "median", round(st.median(v["gflops"] for v in d.values()) / 1e3, 1))
PY
