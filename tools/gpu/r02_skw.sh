# SMSP-balanced DMMA warp map + work-weighted stream-K: parity, f2 / cfg4 / f1 suites (TC_SK_WEIGHTS 0 / 1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "stream_k or subdiv or skinny or cfg4 or edge or epoch or concurrent" 2>&1 | tail -2
for v in 0 1; do
  TC_SK_WEIGHTS=$v timeout 900 python tools/suite.py --family all --no-ttdt > /tmp/a_$v.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
done
python - <<'PY'
import json
a = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/a_0.jsonl")}
b = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/a_1.jsonl")}
for k in a:
    if abs(a[k]["ms"] - b[k]["ms"]) / a[k]["ms"] > 0.02:
        print(f"{k[:34]:34s} w0 {a[k]['ms']*1e3:9.1f}us w1 {b[k]['ms']*1e3:9.1f}us  vs_gemm {a[k]['vs_gemm']:.2f} -> {b[k]['vs_gemm']:.2f}")
PY
cp /tmp/a_1.jsonl gpurun_out/suite_all_skw1.jsonl; cp /tmp/a_0.jsonl gpurun_out/suite_all_skw0.jsonl
