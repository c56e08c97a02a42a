# parity of the skinny / stream-K paths, then the f1 / f2 / baseline suites on the current build
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "skinny or stream_k or subdiv" 2>&1 | tail -2
timeout 1200 python tools/suite.py --family f2 --smtc > gpurun_out/suite_f2_final.jsonl 2>/dev/null
timeout 900 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_f1_final.jsonl 2>/dev/null
timeout 1500 python tools/suite.py --family baseline > gpurun_out/suite_base_final.jsonl 2>/dev/null
python - <<'PY'
import json, statistics
for f in ("f2", "f1", "base"):
    rows = [json.loads(l) for l in open(f"gpurun_out/suite_{f}_final.jsonl")]
    v = [r["vs_gemm"] for r in rows]
    print(f, len(rows), "median vs_gemm", statistics.median(v), "min", min(v))
PY
