# fp32 tcgen05 kernel change: parity of the fp32 paths first, then the cfg4 fp32 suite
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard" > gpurun_out/f32_parity.log 2>&1; tail -2 gpurun_out/f32_parity.log
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" > gpurun_out/f32_full.log 2>&1; tail -2 gpurun_out/f32_full.log
timeout 900 python tools/suite.py --no-ttdt --match "${MATCH:-_f32_}" > gpurun_out/suite_f32_${TAG:-new}.jsonl 2> gpurun_out/suite_f32.err
python - <<'PY'
import json, os
tag = os.environ.get("TAG", "new")
old = {json.loads(l)["config"]: json.loads(l) for l in open("profiles/r02/suite_r02_baseline.jsonl")}
new = [json.loads(l) for l in open(f"gpurun_out/suite_f32_{tag}.jsonl")]
import statistics as st
print("config                                 old_gf    new_gf   ratio  vs_sgemm")
for d in new:
    o = old.get(d["config"], {})
    print(f"{d['config'][:36]:36s} {o.get('gflops',0):9.0f} {d['gflops']:9.0f} {d['gflops']/max(o.get('gflops',1),1):7.3f} {d['vs_gemm']:6.3f}")
print("median new gflops", st.median(d["gflops"] for d in new))
PY
