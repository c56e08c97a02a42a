# skinny kernel: skewed ring layout (TC_SKINNY_SW; auto vs 0) x grid / ring, then parity and ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "skinny or f2_0 or subdiv" 2>&1 | tail -3
for cfg in "-1 4 2" "0 4 2" "-1 2 4" "-1 3 3" "-1 4 3" "-1 2 3"; do set -- $cfg
  TC_SKINNY_SW=$1 TC_SKINNY_CPS=$2 TC_SKINNY_NBUF=$3 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-9]" > /tmp/s.jsonl 2>/dev/null
  python - "$1" "$2" "$3" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"sw={sys.argv[1]} cps={sys.argv[2]} nbuf={sys.argv[3]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_skinny -c 1 -o gpurun_out/f2_00_sw -f \
  python tools/suite.py --family f2 --no-ttdt --match "f2_00" > gpurun_out/ncu_f2_00.log 2>&1
echo ncu $?
