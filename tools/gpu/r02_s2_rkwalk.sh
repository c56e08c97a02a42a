# rank-k v2: strided vs consecutive column-block walks, CTAs per SM in the grid (TC_RANKK_OCC2)
mkdir -p gpurun_out
for rep in 1 2; do
  for occ in 16 64; do
    TC_RANKK_OCC2=$occ timeout 300 python tools/suite.py --no-ttdt --family f1 --only f1_k5_ --reps 10 | sed "s/^/strided$occ /" >> gpurun_out/rkwalk.txt
    TC_RANKK_OCC2=$occ TC_B200_LIB=build_var/tc_consec.so timeout 300 python tools/suite.py --no-ttdt --family f1 --only f1_k5_ --reps 10 | sed "s/^/consec$occ /" >> gpurun_out/rkwalk.txt
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/rkwalk.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    if r["config"].startswith("f1_k5_"): d[v].append((r["ms"], r["hbm_gbs"]))
for v, x in d.items(): print(v, min(x))
PY
