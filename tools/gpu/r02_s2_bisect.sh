# cfg5 bisect of the 0.65% slowdown since checkpoint 2 (same box, alternating builds)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in maxw1 maxw8 maxw16 cur; do
    lib=build_var/tc_$v.so; [ $v = cur ] && lib=""
    TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --only cfg5 --reps 2 | sed "s/^/$v /" >> gpurun_out/bisect3.txt 2>&1
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/bisect3.txt"):
    v, j = l.split(" ", 1)
    try: d[v].append(json.loads(j)["ms"])
    except Exception: pass
for v, x in d.items(): print(v, min(x), x)
PY
