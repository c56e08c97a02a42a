# fp32: A's 16-byte M vectors in the N = 256 form (TC_UMMA_FORM=256) vs the N = 128 form (default
# for those cases) and vs N = 256 without them (TC_UMMA_AM=0)
mkdir -p gpurun_out
TC_UMMA_FORM=256 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32_vector or f32_pair or f32_loader or guard_bands_f32" 2>&1 | tail -1
timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/am_default.jsonl 2>/dev/null
TC_UMMA_FORM=256 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/am_256.jsonl 2>/dev/null
TC_UMMA_FORM=256 TC_UMMA_AM=0 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/am_256_noam.jsonl 2>/dev/null
SWEEP_DTYPE=f32 TC_UMMA_FORM=256 timeout 600 python tools/f32_size_sweep.py 2>/dev/null | cut -c1-120
python - <<'PY'
import json, math, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
R = {f: load(f"gpurun_out/am_{f}.jsonl") for f in ("default", "256", "256_noam")}
for k in R["default"]:
    print(f"{k[:34]:34s} " + " ".join(f"{R[f][k]['gflops']/1e3:6.1f}" for f in R) + f"  a_vec_m={R['default'][k]['a_vec_m']}")
for f, d in R.items():
    v = [x["gflops"] for x in d.values()]
    print(f, "median", round(st.median(v)/1e3, 1), "geomean", round(math.exp(sum(math.log(x) for x in v)/len(v))/1e3, 1))
PY
