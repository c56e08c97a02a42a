# skinny kernel grid / ring sweep on the HBM-bound fig:bench strings (N = K = 32) and one N = K = 76
mkdir -p gpurun_out
for cfg in "3 3" "2 5" "4 2" "5 2" "2 4" "3 2" "6 2"; do set -- $cfg
  TC_SKINNY_CPS=$1 TC_SKINNY_NBUF=$2 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-4]" > /tmp/s.jsonl 2>/dev/null
  python - "$1" "$2" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"cps={sys.argv[1]} nbuf={sys.argv[2]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
