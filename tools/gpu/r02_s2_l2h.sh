# skinny kernel: L2 prefetch hint of the X copies (default / L2::128B / L2::256B)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in def l2h128 l2h256; do
    lib=build_var/tc_$v.so; [ $v = def ] && lib=""
    TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --family f2 --only f2_0 --reps 10 | sed "s/^/$v /" >> gpurun_out/l2h.txt
    TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --family f2 --only f2_1 --reps 10 | sed "s/^/$v /" >> gpurun_out/l2h.txt
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/l2h.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append((r["ms"], r["hbm_gbs"]))
for c, x in d.items():
    print(c[:28].ljust(28), "  ".join("%s %.4f (%5.0f)" % (k, min(v)[0], min(v)[1]) for k, v in x.items()))
PY
