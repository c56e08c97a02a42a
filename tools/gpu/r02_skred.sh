# stream-K accumulation through red.global.add.f64 (default) vs load-add-store (-DTC_SK_RED=0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "stream_k or epoch or concurrent or fresh or cfg4_scaled or cfg5_scaled" 2>&1 | tail -2
for v in def nored; do
  if [ $v = def ]; then LIB=""; else LIB=$PWD/build_var/lib_$v.so; fi
  echo "== $v"
  TC_B200_LIB=$LIB SWEEP_DTYPE=f64 SWEEP_SIZES=512x512x512,768x768x768,1024x1024x1024,256x256x65536 timeout 300 python tools/f32_size_sweep.py | cut -c1-130
  TC_B200_LIB=$LIB timeout 900 python tools/suite.py --family all --no-ttdt > /tmp/a_$v.jsonl 2>/dev/null
done
python - <<'PY'
import json
a = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/a_nored.jsonl")}
b = {json.loads(l)["config"]: json.loads(l) for l in open("/tmp/a_def.jsonl")}
for k in a:
    if abs(a[k]["ms"] - b[k]["ms"]) / a[k]["ms"] > 0.02:
        print(f"{k[:34]:34s} nored {a[k]['ms']*1e3:9.1f}us red {b[k]['ms']*1e3:9.1f}us  vs_gemm {a[k]['vs_gemm']:.2f} -> {b[k]['vs_gemm']:.2f}")
PY
cp /tmp/a_def.jsonl gpurun_out/suite_all_skred.jsonl
