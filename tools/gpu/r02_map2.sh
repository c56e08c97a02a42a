# attribution of the one-line gathers: K gathers (k), row gathers (r), both, neither
mkdir -p gpurun_out
for M in kr krb k 0; do TC_UMMA_MAP=$M timeout 900 python tools/suite.py --no-ttdt --match "_f32_" > gpurun_out/map2_$M.jsonl 2>/dev/null; done
python - <<'PY'
import json, statistics as st
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
R = {m: load(f"gpurun_out/map2_{m}.jsonl") for m in ("kr", "krb", "k", "0")}
print("config                               kr    krb      k      0   (TF/s)  a_vec_m b_vec_k")
for k, d in R["0"].items():
    print(f"{k[:34]:34s} " + " ".join(f"{R[m][k]['gflops']/1e3:6.1f}" for m in ("kr", "krb", "k", "0")) + f"   {d['a_vec_m']} {d['b_vec_k']}")
for m, d in R.items(): print(m, "median", round(st.median(v["gflops"] for v in d.values()) / 1e3, 1))
PY
