# two-level P sub-division (default) vs one level (TC_KBLOCK=flat) on the fig:bench strings with K sub-division
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "subdiv or f2 or cfg4_05" 2>&1 | tail -2
for v in flat two; do
  TC_KBLOCK=$v timeout 600 python tools/suite.py --family f2 --no-ttdt > /tmp/s_$v.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  TC_KBLOCK=$v timeout 600 python tools/suite.py --only cfg4 --no-ttdt > /tmp/c_$v.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
done
python - <<'PY'
import json
for fam in ("s", "c"):
    a = {json.loads(l)["config"]: json.loads(l) for l in open(f"/tmp/{fam}_flat.jsonl")}
    b = {json.loads(l)["config"]: json.loads(l) for l in open(f"/tmp/{fam}_two.jsonl")}
    for k in a:
        if abs(a[k]["ms"] - b[k]["ms"]) / a[k]["ms"] > 0.02:
            print(f"{k[:34]:34s} flat {a[k]['ms']*1e3:9.1f}us two {b[k]['ms']*1e3:9.1f}us  vs_gemm {a[k]['vs_gemm']:.2f} -> {b[k]['vs_gemm']:.2f}")
PY
cp /tmp/s_two.jsonl gpurun_out/suite_f2_kblock2.jsonl; cp /tmp/s_flat.jsonl gpurun_out/suite_f2_kblock1.jsonl
timeout 600 ncu --set full --clock-control none -k regex:tc_ -c 1 -o gpurun_out/f2_16_k2 -f \
  python tools/suite.py --family f2 --no-ttdt --match "f2_16" > /dev/null 2>&1; echo ncu $?
