# fp32 tcgen05 register path (gather mode 4) vs the cp.async gathers (TC_UMMA_RP=0): parity of
# every fp32 path first, then the cfg4 fp32 suite both ways on the same box
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_ablation.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard or Stream or epoch or ablation or forced" > gpurun_out/rp_parity.log 2>&1; tail -3 gpurun_out/rp_parity.log
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f32" > gpurun_out/rp_full.log 2>&1; tail -2 gpurun_out/rp_full.log
timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/suite_rp1.jsonl 2> gpurun_out/suite_rp.err
TC_UMMA_RP=0 timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/suite_rp0.jsonl 2>> gpurun_out/suite_rp.err
for F in 128 256; do TC_UMMA_FORM=$F timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/suite_rp1_f$F.jsonl 2>> gpurun_out/suite_rp.err; done
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
a, b = load("gpurun_out/suite_rp0.jsonl"), load("gpurun_out/suite_rp1.jsonl")
f1, f2 = load("gpurun_out/suite_rp1_f128.jsonl"), load("gpurun_out/suite_rp1_f256.jsonl")
print("config                              rp0_gf   rp1_gf  ratio   f128   f256  vs_sgemm")
for k in a:
    print(f"{k[:34]:34s} {a[k]['gflops']:8.0f} {b[k]['gflops']:8.0f} {b[k]['gflops']/a[k]['gflops']:6.3f} {f1[k]['gflops']:7.0f} {f2[k]['gflops']:7.0f} {b[k]['vs_gemm']:6.3f}")
for n, d in (("rp0", a), ("rp1", b), ("f128", f1), ("f256", f2)):
    print(n, "median", st.median(v["gflops"] for v in d.values()))
PY
