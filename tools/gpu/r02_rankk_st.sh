# rank-k kernel: C stores with st.global.L1::no_allocate (default build) vs plain (variant library)
for v in def rk0; do
  if [ $v = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$v.so; fi
  TC_B200_LIB=$LIB timeout 300 python tools/suite.py --family f1 --no-ttdt > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$v" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"{sys.argv[1]} " + "  ".join(f"{r['config'][:6]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:5.0f}GB/s" for r in rows))
PY
done
timeout 600 python -m pytest tests -m gpu -x -q -k "rankk or skinny" 2>&1 | tail -2
