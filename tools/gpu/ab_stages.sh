# parity + per-config suite with the default build, then the cfg4 fp32 suite with a 4-stage fp32 variant
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python tools/suite.py --no-ttdt > gpurun_out/suite_default.jsonl 2> gpurun_out/suite_default.err
TC_LIB_OUT=/tmp/tc_s4.so TC_NVCC_EXTRA="-DTC_STAGES_F32=4" python paper_1607_00291_b200/_build.py > /dev/null 2>&1
TC_B200_LIB=/tmp/tc_s4.so timeout 600 python tools/suite.py --no-ttdt --only cfg4 > gpurun_out/suite_s4.jsonl 2>&1
python - <<'PY'
import json
def load(p):
    return {d["config"]: d for d in map(json.loads, open(p)) }
a=load("gpurun_out/suite_default.jsonl"); b=load("gpurun_out/suite_s4.jsonl")
for k,d in a.items():
    o=b.get(k,{})
    print(f"{k[:34]:34s} {d['gflops']:9.0f} gemm {d['gemm_gflops']:9.0f} r={d['vs_gemm']:.3f}  s4 r={o.get('vs_gemm')}")
PY
