# fp32 form per case after the round-2 gather changes: default vs N = 128 vs N = 256 forced
mkdir -p gpurun_out
for F in default 128 256; do
  if [ $F = default ]; then E=""; else E="TC_UMMA_FORM=$F"; fi
  env $E timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/forms2_$F.jsonl 2>/dev/null
done
python - <<'PY'
import json, statistics as st, sys, os
sys.path.insert(0, os.getcwd())
import torch, workloads as W, paper_1607_00291_b200 as tc
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
R = {f: load(f"gpurun_out/forms2_{f}.jsonl") for f in ("default", "128", "256")}
print("config                              dflt   f128   f256  modes(A vec/pair, B vec/pair)")
for i in range(20):
    case = W.cfg4(i, torch.float32)
    k = case.name
    shapes=[case.shape(l) for l in (case.lab_a, case.lab_b, case.lab_c)]
    p = tc.Plan(case.spec, torch.float32, shapes, [W.colmajor_strides(s) for s in shapes])
    print(f"{k[:34]:34s} " + " ".join(f"{R[f][k]['gflops']/1e3:6.1f}" for f in ("default", "128", "256")))
for f, d in R.items(): print(f, "median", round(st.median(v["gflops"] for v in d.values())/1e3, 1))
PY
