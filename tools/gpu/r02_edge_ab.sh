# A/B in one call: default build (edge skipping) vs -DTC_DMMA_EDGE=0, cfg4 fp64 + f2 edge-heavy
mkdir -p gpurun_out
TC_LIB_OUT=/tmp/tc_noedge.so TC_NVCC_EXTRA="-DTC_DMMA_EDGE=0" python paper_1607_00291_b200/_build.py > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; exit 1; }
for r in 1 2; do
  timeout 900 python tools/suite.py --family all --no-ttdt --match "cfg4_.._f64|f2_(05|09|11|15|16|17|18)" > gpurun_out/eab_edge_$r.jsonl 2>/dev/null
  TC_B200_LIB=/tmp/tc_noedge.so timeout 900 python tools/suite.py --family all --no-ttdt --match "cfg4_.._f64|f2_(05|09|11|15|16|17|18)" > gpurun_out/eab_noedge_$r.jsonl 2>/dev/null
done
python - <<'PY'
import json
def load(p): return {json.loads(l)["config"]: json.loads(l) for l in open(p)}
E = [load(f"gpurun_out/eab_edge_{r}.jsonl") for r in (1, 2)]
N = [load(f"gpurun_out/eab_noedge_{r}.jsonl") for r in (1, 2)]
print("config                              edge1  edge2  noedge1 noedge2 (TF/s)")
for k in E[0]:
    print(f"{k[:34]:34s} {E[0][k]['gflops']/1e3:6.2f} {E[1][k]['gflops']/1e3:6.2f} {N[0][k]['gflops']/1e3:6.2f} {N[1][k]['gflops']/1e3:6.2f}")
PY
