# Round-2 session-2 checkpoint: smoke, the whole GPU suite, bench (N=1), reference arm, baseline suite
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/ck_smoke.log 2>&1; tail -3 gpurun_out/ck_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/ck_gputest.log 2>&1; tail -4 gpurun_out/ck_gputest.log
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; cut -c1-300 gpurun_out/ck_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/ck_ref.json 2> gpurun_out/ck_ref.err; cut -c1-200 gpurun_out/ck_ref.json
timeout 1500 python tools/suite.py --family baseline > gpurun_out/suite_base_s2.jsonl 2>/dev/null
python - <<'PY'
import json, statistics
rows = [json.loads(l) for l in open("gpurun_out/suite_base_s2.jsonl")]
f32 = [r["gflops"] / 1e3 for r in rows if r["dtype"] == "float32"]
print("cfg4 fp32 TF/s median", statistics.median(f32), "geomean", statistics.geometric_mean(f32))
PY
