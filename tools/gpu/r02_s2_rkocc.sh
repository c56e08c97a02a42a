# rank-k v2 with consecutive walks: CTAs per SM in the grid (TC_RANKK_OCC2), parity of the kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "rankk" > gpurun_out/rko_tests.log 2>&1; tail -2 gpurun_out/rko_tests.log
for rep in 1 2; do
  for occ in 8 16 32 64 128 256; do
    TC_RANKK_OCC2=$occ timeout 300 python tools/suite.py --no-ttdt --family f1 --only f1_k5_ --reps 10 | sed "s/^/occ$occ /" >> gpurun_out/rkocc.txt
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/rkocc.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    if r["config"].startswith("f1_k5_"): d[v].append((r["ms"], r["hbm_gbs"], r["vs_gemm"]))
for v, x in d.items(): print(v, min(x))
PY
