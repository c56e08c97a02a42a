timeout 1200 python -m pytest tests -m gpu -x -q -k "stream_k or epoch or concurrent or fresh or cfg4_scaled or cfg5_scaled or f2_ or skinny" 2>&1 | tail -2
SWEEP_DTYPE=f64 SWEEP_SIZES=512x512x512,768x768x768,1024x1024x1024,256x256x65536 timeout 300 python tools/f32_size_sweep.py | cut -c1-130
bash tools/gpu/r02_skred2.sh
timeout 900 python tools/suite.py --only cfg --no-ttdt > /tmp/cfg_def.jsonl 2>/dev/null
TC_B200_LIB=$PWD/build_var/lib_nored.so timeout 900 python tools/suite.py --only cfg --no-ttdt > /tmp/cfg_nored.jsonl 2>/dev/null
python - <<'PY'
import json
a = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/cfg_nored.jsonl")}
b = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/cfg_def.jsonl")}
for k in a:
    if abs(a[k]["ms"] - b[k]["ms"]) / a[k]["ms"] > 0.02:
        print(f"{k[:34]:34s} nored {a[k]['ms']*1e3:9.1f}us red {b[k]['ms']*1e3:9.1f}us")
PY
