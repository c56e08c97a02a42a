# FP64 pipe mix calibration + skinny kernel at 3 CTAs per SM (register cap, variant library)
mkdir -p gpurun_out tools/calib/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/calib/bin/fp64_mix tools/calib/fp64_mix.cu && timeout 120 tools/calib/bin/fp64_mix | tee gpurun_out/calib_fp64_mix.jsonl
for cfg in "def 4 2" "minb3 3 2" "minb3 3 3" "minb3 6 2" "minb3 3 4"; do set -- $cfg
  if [ $1 = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$1.so; fi
  TC_B200_LIB=$LIB TC_SKINNY_CPS=$2 TC_SKINNY_NBUF=$3 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_0[0-4]" > /tmp/s.jsonl 2>/dev/null
  python - "$1" "$2" "$3" <<'PY'
import json, sys
rows = [json.loads(l) for l in open("/tmp/s.jsonl")]
print(f"lib={sys.argv[1]} cps={sys.argv[2]} nbuf={sys.argv[3]} " + "  ".join(f"{r['config'][:5]} {r['ms']*1e3:6.1f}us {r['hbm_gbs']:6.0f}GB/s" for r in rows))
PY
done
