# Round-2 session-3 final baseline suite on the final build (cfg1-cfg5, cfg4 fp64 + fp32, TTDT comparator)
mkdir -p gpurun_out
timeout 1100 python tools/suite.py --family baseline > gpurun_out/suite_r02s3_baseline_ck10.jsonl 2>gpurun_out/suite_base.err
python - <<'PY'
import json, statistics
rows = [json.loads(l) for l in open("gpurun_out/suite_r02s3_baseline_ck10.jsonl")]
for dt in ("float64", "float32"):
    r = [x for x in rows if x.get("dtype") == dt and x["config"].startswith("cfg4")]
    print(dt, len(r), "cfg4 median TF/s", statistics.median(x["gflops"] for x in r) / 1e3, "median vs_gemm", statistics.median(x["vs_gemm"] for x in r), "min", min(x["vs_gemm"] for x in r))
PY
