for st in 2 3 4 6; do
  TC_SKINNY_WS_STAGES=$st timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-6]|f2_1[234]" > /tmp/s.jsonl 2>/dev/null
  python - "$st" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"st={sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}" for r in rows))
PY
done
for v in 0 1; do
  TC_SKINNY_WS_CG=1 TC_SKINNY_WS_STAGES=2 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[013]" > /tmp/s.jsonl 2>/dev/null
done
python - <<'PY'
import json
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print("cg1 st2 " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}" for r in rows))
PY
