# rank-k version 3 (FP64 tensor cores, K <= 32): parity, then f1 timings v2 / v3 / tile kernel
timeout 1200 python -m pytest tests -m gpu -x -q -k "rankk" 2>&1 | tail -2
for cfg in "2 1 1" "3 1 1" "2 0 0"; do set -- $cfg
  TC_RANKK_V=$1 TC_RANKK=$2 TC_RANKK16=$3 timeout 600 python tools/suite.py --family f1 --no-ttdt > /tmp/s.jsonl 2>/dev/null
  python - "$1" "$2" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"v={sys.argv[1]} rankk={sys.argv[2]} " + "  ".join(f"{r['config'][:6]} {r['ms']*1e3:7.1f}us {r['hbm_gbs']:5.0f}" for r in rows))
PY
done
for occ in 16 32 128; do
  TC_RANKK_V=3 TC_RANKK_OCC2=$occ timeout 600 python tools/suite.py --family f1 --no-ttdt --match "f1_k(5|16|32)_" > /tmp/s.jsonl 2>/dev/null
  python - "$occ" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"v3 occ={sys.argv[1]} " + "  ".join(f"{r['config'][:6]} {r['ms']*1e3:7.1f}us {r['hbm_gbs']:5.0f}" for r in rows))
PY
done
