# cfg4 fp32: the kernel's form choice vs each form forced (N = 256 now with vector gathers too)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "f32 or guard" > gpurun_out/forms_parity.log 2>&1; tail -2 gpurun_out/forms_parity.log
for F in default 128 256; do
  if [ $F = default ]; then E=""; else E="TC_UMMA_FORM=$F"; fi
  env $E timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/suite_form_$F.jsonl 2>> gpurun_out/suite_form.err
done
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
R = {f: load(f"gpurun_out/suite_form_{f}.jsonl") for f in ("default", "128", "256")}
print("config                               default      f128      f256  a_vec_m b_vec_k")
for k, d in R["default"].items():
    print(f"{k[:36]:36s} {d['gflops']:9.0f} {R['128'][k]['gflops']:9.0f} {R['256'][k]['gflops']:9.0f}  {d['a_vec_m']} {d['b_vec_k']}")
for f, d in R.items():
    print(f, "median", st.median(v["gflops"] for v in d.values()))
PY
