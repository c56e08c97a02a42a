# fp64 DMMA kernel: stream-K threshold for the partial wave (TC_WS_DPPCT; default 88)
mkdir -p gpurun_out
for P in 88 95 101; do TC_WS_DPPCT=$P timeout 600 python tools/suite.py --no-ttdt --match "cfg4_.._f64" > gpurun_out/dp_$P.jsonl 2>/dev/null; done
python - <<'PY'
import json, statistics as st
R = {p: {json.loads(l)["config"]: json.loads(l) for l in open(f"gpurun_out/dp_{p}.jsonl")} for p in (88, 95, 101)}
print("config                              dp88    dp95   dp101   (TF/s)  tiles")
for k, d in R[88].items():
    m, n, kk = d["mnk"]
    t = ((m + 127) // 128) * ((n + 127) // 128)
    print(f"{k[:34]:34s} {d['gflops']/1e3:6.2f} {R[95][k]['gflops']/1e3:6.2f} {R[101][k]['gflops']/1e3:6.2f}   {t} ({t/148:.2f} waves)")
for p, d in R.items(): print(p, "median", st.median(v["gflops"] for v in d.values()), "min", min(v["gflops"] for v in d.values()))
PY
