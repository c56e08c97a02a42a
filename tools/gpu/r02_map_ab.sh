# DMMA consumer warp map A/B (default SMSP-balanced map vs -DTC_DMMA_OLDMAP) on cfg5 and cfg2-4 fp64
for rep in 1 2; do for v in def oldmap; do
  if [ $v = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$v.so; fi
  TC_B200_LIB=$LIB timeout 600 python tools/suite.py --only cfg5 --no-ttdt --reps 3 > /tmp/s.jsonl 2>/dev/null
  TC_B200_LIB=$LIB timeout 600 python tools/suite.py --only cfg4 --no-ttdt > /tmp/c.jsonl 2>/dev/null
  python - "$v" <<'PY'
import json, sys, statistics
r = [json.loads(l) for l in open("/tmp/s.jsonl")]
c = [json.loads(l) for l in open("/tmp/c.jsonl") if "f64" in json.loads(l)["config"]]
print(sys.argv[1], "cfg5", r[0]["gflops"], "cfg4 f64 median", statistics.median(x["gflops"] for x in c))
PY
done; done
