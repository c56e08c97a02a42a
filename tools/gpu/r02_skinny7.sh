# skinny: 16-byte X copies (TC_SKINNY_VEC) in the warp-specialised form: parity, sweep, ablation, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "skinny" 2>&1 | tail -3
for cfg in "0 6" "1 6" "1 4" "1 8"; do set -- $cfg
  TC_SKINNY_VEC=$1 TC_SKINNY_WS_STAGES=$2 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-4]" > /tmp/s.jsonl 2>/tmp/s.err || tail -3 /tmp/s.err
  python - "$1" "$2" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"vec={sys.argv[1]} st={sys.argv[2]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
TC_SKINNY_VEC=1 timeout 300 python tools/skinny_layouts.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_skinny -c 1 -o gpurun_out/f2_00_vec -f \
  python tools/suite.py --family f2 --no-ttdt --match "f2_00" > gpurun_out/ncu_f2_00_vec.log 2>&1
echo ncu $?
