# fp32 gather mode 12 (B along N by shifted 16-byte vectors): parity, modes, cfg4 A/B vs elements
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shifted or f32_vector or f32_pair or cfg4_scaled_f32 or guard_bands_f32" > gpurun_out/sh_tests.log 2>&1; tail -3 gpurun_out/sh_tests.log
TC_UMMA_DEBUG=1 timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 1 2>&1 | grep -E "tc_umma|f32" | cut -c1-120 > gpurun_out/sh_modes.txt
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 >> gpurun_out/sh_on.jsonl 2>&1
  TC_UMMA_SHIFT=0 timeout 600 python tools/suite.py --no-ttdt --only cfg4 --reps 5 >> gpurun_out/sh_off.jsonl 2>&1
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
on, off = load("gpurun_out/sh_on.jsonl"), load("gpurun_out/sh_off.jsonl")
for k in on:
    a, b = min(on[k]), min(off[k])
    print(k[:32].ljust(32), "shift %.4f elem %.4f  %.3fx" % (a, b, b / a))
PY
