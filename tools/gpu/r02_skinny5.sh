# skinny warp-specialised form: parity, then WS on/off x consumer groups x stages on f2_00-04, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "skinny" 2>&1 | tail -3
for cfg in "0 2 0" "1 2 0" "1 1 0" "1 2 4" "1 2 6" "1 1 4"; do set -- $cfg
  TC_SKINNY_WS=$1 TC_SKINNY_WS_CG=$2 TC_SKINNY_WS_STAGES=$3 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-4]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$1" "$2" "$3" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"ws={sys.argv[1]} cg={sys.argv[2]} st={sys.argv[3]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_skinny -c 1 -o gpurun_out/f2_00_ws -f \
  python tools/suite.py --family f2 --no-ttdt --match "f2_00" > gpurun_out/ncu_f2_00_ws.log 2>&1
echo ncu $?
