# skinny kernel component ablation (TC_SKINNY_DBG: 1 no MMA, 2 no X loads, 4 no stores) on f2_00-04
mkdir -p gpurun_out
for dbg in 0 1 2 4 3 5 6; do
  TC_SKINNY_DBG=$dbg timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-4]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$dbg" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"dbg={sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us" for r in rows))
PY
done
