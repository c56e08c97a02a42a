# fp32 tcgen05 kernel: stream-K threshold (TC_UMMA_DPPCT, default 70) on cfg4 fp32
mkdir -p gpurun_out
for rep in 1 2; do
  for p in 70 85 101; do
    TC_UMMA_DPPCT=$p timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 2>/dev/null | grep float32 | sed "s/^/$p /" >> gpurun_out/ummask2.txt
  done
  : TC_UMMA_SK=0 timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 2>/dev/null | grep float32 | sed "s/^/nosk /" >> gpurun_out/ummask2.txt
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/ummask2.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append(r["ms"])
g = collections.defaultdict(list)
for c, x in d.items():
    b = min(x["70"])
    line = []
    for p in ("85", "101"):
        g[p].append(b / min(x[p])); line.append("%s %.3f" % (p, b / min(x[p])))
    print(c[:30].ljust(30), "70 %.4f ms " % b, " ".join(line))
for p, v in g.items(): print("speedup vs 70:", p, "geomean %.4f min %.3f max %.3f" % (statistics.geometric_mean(v), min(v), max(v)))
PY
