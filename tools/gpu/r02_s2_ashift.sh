# fp32 gather mode 13 (A along M by shifted vectors with bulk copies): parity, modes, cfg4 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shifted or f32_vector or f32_pair or cfg4_scaled_f32 or guard_bands_f32" > gpurun_out/as_tests.log 2>&1; tail -3 gpurun_out/as_tests.log
TC_UMMA_DEBUG=1 timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 1 2>&1 | grep -E "tc_umma" | uniq > gpurun_out/as_modes.txt
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 >> gpurun_out/as_on.jsonl 2>&1
  TC_UMMA_ASHIFT=0 timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 >> gpurun_out/as_off.jsonl 2>&1
done
python - <<'PY'
import json, collections
def load(f):
    d = collections.defaultdict(list)
    for l in open(f):
        try: r = json.loads(l)
        except Exception: continue
        if r["dtype"] == "float32": d[r["config"]].append(r["ms"])
    return d
on, off = load("gpurun_out/as_on.jsonl"), load("gpurun_out/as_off.jsonl")
for k in on:
    a, b = min(on[k]), min(off[k])
    print(k[:32].ljust(32), "ashift %.4f off %.4f  %.3fx" % (a, b, b / a))
PY
