# Skinny kernel: C run length of the sub-division (TC_SKINNY_BV = 8 default | 16 | 32) on the
# fig:bench skinny strings; parity of the override first
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "skinny_run" > gpurun_out/bv_parity.log 2>&1; tail -2 gpurun_out/bv_parity.log
for rep in 1 2; do
for bv in 8 BU16 BU32 BU4; do
  if [ "${bv#BU}" != "$bv" ]; then export TC_SKINNY_BU=${bv#BU}; else unset TC_SKINNY_BU; fi; timeout 300 python tools/suite.py --family f2 --match 'f2_0[0-4]' --no-ttdt --reps 20 > gpurun_out/bv_$bv.$rep.jsonl 2>/dev/null
  python - $bv $rep <<'PY'
import json, sys
for l in open(f"gpurun_out/bv_{sys.argv[1]}.{sys.argv[2]}.jsonl"):
    r = json.loads(l)
    print("bv", sys.argv[1], r["config"][:20], "%.1f us" % (r["ms"] * 1e3), "%.0f GB/s" % r["hbm_gbs"], "vs_gemm %.3f" % r["vs_gemm"])
PY
done
done
