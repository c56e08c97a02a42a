# skinny warp-specialised form: C store cache hints (variant libraries, -DTC_SKINNY_STHINT)
for v in def st1 st2 st3; do
  if [ $v = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$v.so; fi
  TC_B200_LIB=$LIB timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[013]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$v" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"{sys.argv[1]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
  TC_B200_LIB=$LIB TC_SKINNY_DBG=3 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_00" 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('  stores only f2_00', round(r['ms']*1e3,1), 'us')"
done
