mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "skinny_warp or skinny_vec" 2>&1 | tail -2
for v in 0 1; do
  TC_SKINNY_VEC=$v timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[013]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$v" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"vec={sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
TC_SKINNY_VEC=1 timeout 300 python tools/skinny_layouts.py
