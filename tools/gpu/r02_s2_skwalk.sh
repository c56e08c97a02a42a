# skinny kernel (warp-specialised form): consecutive vs strided block ranges per CTA; parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "skinny or f2" > gpurun_out/skw_tests.log 2>&1; tail -2 gpurun_out/skw_tests.log
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --family f2 --reps 10 | sed "s/^/consec /" >> gpurun_out/skwalk.txt
  TC_B200_LIB=build_var/tc_strided.so timeout 600 python tools/suite.py --no-ttdt --family f2 --reps 10 | sed "s/^/strided /" >> gpurun_out/skwalk.txt
done
python - <<'PY'
import json, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/skwalk.txt"):
    v, j = l.split(" ", 1)
    try: r = json.loads(j)
    except Exception: continue
    d[r["config"]][v].append((r["ms"], r["hbm_gbs"], r["vs_gemm"]))
for c, x in d.items():
    a, b = min(x["consec"]), min(x["strided"])
    print(c[:30].ljust(30), "consec %.4f ms %6.0f GB/s %.3f | strided %.4f ms %6.0f GB/s %.3f | %.3fx" % (a + b + (b[0] / a[0],)))
PY
