# kernel-parameter size A/B on cfg4 (fp32 tcgen05 and fp64 DMMA kernels): Sched with 16 vs 1 weights
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 | sed "s/^/cur /" >> gpurun_out/param.txt 2>&1
  TC_B200_LIB=build_var/tc_maxw1.so timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 | sed "s/^/w1 /" >> gpurun_out/param.txt 2>&1
done
python - <<'PY'
import json, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/param.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append(r["ms"])
import statistics
rat = {"float32": [], "float64": []}
for c, x in d.items():
    r = min(x["cur"]) / min(x["w1"]); rat["float32" if "f32" in c else "float64"].append(r)
    print(c[:32].ljust(32), "cur %.4f w1 %.4f  cur/w1 %.3f" % (min(x["cur"]), min(x["w1"]), r))
for k, v in rat.items(): print(k, "geomean cur/w1", statistics.geometric_mean(v))
PY
