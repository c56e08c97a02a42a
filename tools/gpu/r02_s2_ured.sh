# fp32 tcgen05 kernel: stream-K fix-ups by red.global.add.f32 vs load-add-store; parity first
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "f32 and (stream_k or guard or cfg4 or vector or pair or shifted or bias)" > gpurun_out/ur_tests.log 2>&1; tail -2 gpurun_out/ur_tests.log
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 2>/dev/null | grep float32 | sed "s/^/red /" >> gpurun_out/ured.txt
  TC_B200_LIB=build_var/tc_nored.so timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 2>/dev/null | grep float32 | sed "s/^/rmw /" >> gpurun_out/ured.txt
  SWEEP_SIZES=512x512x512,768x768x768,1024x1024x1024,1536x1536x1536,256x256x65536,4096x4096x64 timeout 600 python tools/f32_size_sweep.py 2>/dev/null | sed "s/^/red /" >> gpurun_out/ured_sw.txt
  SWEEP_SIZES=512x512x512,768x768x768,1024x1024x1024,1536x1536x1536,256x256x65536,4096x4096x64 TC_B200_LIB=build_var/tc_nored.so timeout 600 python tools/f32_size_sweep.py 2>/dev/null | sed "s/^/rmw /" >> gpurun_out/ured_sw.txt
done
python - <<'PY'
import json, collections, statistics
d = collections.defaultdict(lambda: collections.defaultdict(list))
for f, key in (("gpurun_out/ured.txt", "config"), ("gpurun_out/ured_sw.txt", "mnk")):
    for l in open(f):
        v, j = l.split(" ", 1)
        try: r = json.loads(j)
        except Exception: continue
        d[str(r[key])][v].append(r["ms"])
g = []
for c, x in d.items():
    r = min(x["rmw"]) / min(x["red"]); g.append(r)
    print(c[:32].ljust(32), "rmw %.4f red %.4f  %.3fx" % (min(x["rmw"]), min(x["red"]), r))
print("geomean", statistics.geometric_mean(g))
PY
