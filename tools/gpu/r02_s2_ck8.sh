# Round-2 session-2 checkpoint 8: smoke, whole GPU suite, bench (N=1), reference arm, the three
# suites (baseline with TTDT, f1, f2 with the SMTC ablation), the bench launch list
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/ck_smoke.log 2>&1; tail -3 gpurun_out/ck_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/ck_gputest.log 2>&1; tail -4 gpurun_out/ck_gputest.log
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; cut -c1-300 gpurun_out/ck_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/ck_ref.json 2> gpurun_out/ck_ref.err; cut -c1-200 gpurun_out/ck_ref.json
timeout 1500 python tools/suite.py --family baseline > gpurun_out/suite_base_ck8.jsonl 2>/dev/null
timeout 1200 python tools/suite.py --family f2 --smtc > gpurun_out/suite_f2_ck8.jsonl 2>/dev/null
timeout 900 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_f1_ck8.jsonl 2>/dev/null
python - <<'PY'
import json, statistics
for f in ("base", "f1", "f2"):
    rows = [json.loads(l) for l in open(f"gpurun_out/suite_{f}_ck8.jsonl")]
    v = [r["vs_gemm"] for r in rows]
    print(f, len(rows), "median vs_gemm", statistics.median(v), "min", min(v))
rows = [json.loads(l) for l in open("gpurun_out/suite_base_ck8.jsonl")]
f32 = [r["gflops"] / 1e3 for r in rows if r["dtype"] == "float32"]
f64 = [r["gflops"] / 1e3 for r in rows if r["dtype"] == "float64" and r["config"].startswith("cfg4")]
print("cfg4 fp32 TF/s median", statistics.median(f32), "geomean", statistics.geometric_mean(f32), "min", min(f32))
print("cfg4 fp64 TF/s median", statistics.median(f64), "min", min(f64))
PY
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench_r02s2c.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ck_ncu.log 2>&1
echo "ncu rc=$?"
python tools/summarize_launches.py gpurun_out/launches_bench_r02s2c.csv > gpurun_out/launches_bench_r02s2c.summary.txt; head -20 gpurun_out/launches_bench_r02s2c.summary.txt
