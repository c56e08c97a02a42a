# re-measure the DMMA kernel's stream-K threshold (partial wave >= DPPCT% full runs
# data-parallel) now that the fix-ups add at L2 (red.global.add): fp64 baseline, f1, f2
mkdir -p gpurun_out
for rep in 1 2; do
  for p in 88 95 101; do
    TC_WS_DPPCT=$p timeout 900 python tools/suite.py --no-ttdt --family baseline --only cfg4 --reps 5 2>/dev/null | grep float64 | sed "s/^/$p /" >> gpurun_out/dppct.txt
    TC_WS_DPPCT=$p timeout 900 python tools/suite.py --no-ttdt --family f2 --reps 3 2>/dev/null | sed "s/^/$p /" >> gpurun_out/dppct.txt
    TC_WS_DPPCT=$p timeout 900 python tools/suite.py --no-ttdt --family f1 --reps 3 2>/dev/null | sed "s/^/$p /" >> gpurun_out/dppct.txt
  done
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/dppct.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append(r["ms"])
g = collections.defaultdict(list)
for c, x in d.items():
    b = min(x["88"])
    line = []
    for p in ("95", "101"):
        if p in x:
            g[p].append(b / min(x[p])); line.append("%s %.3f" % (p, b / min(x[p])))
    print(c[:30].ljust(30), "88 %.4f ms  " % b, "  ".join(line))
for p, v in g.items(): print("speedup vs 88:", p, "geomean %.4f min %.3f max %.3f" % (statistics.geometric_mean(v), min(v), max(v)))
PY
