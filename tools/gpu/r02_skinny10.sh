# skinny warp-specialised form for the larger resident operands (TC_SKINNY_WS_BIG): parity + f2 timings
timeout 900 python -m pytest tests -m gpu -x -q -k "skinny" 2>&1 | tail -2
for v in 0 1; do
  TC_SKINNY_WS_BIG=$v timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-6]|f2_1[234]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$v" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"big={sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['vs_gemm']:.2f}" for r in rows))
PY
done
for st in 2 3; do
  TC_SKINNY_WS_STAGES=$st timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[246]|f2_1[234]" > /tmp/s.jsonl 2>/dev/null
  python - "$st" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"st={sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['vs_gemm']:.2f}" for r in rows))
PY
done
