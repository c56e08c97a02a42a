# fp32 A/B: default build vs -DTC_FFMA_PAIRK=0, plus stream-K off and DMMA fp32 on the default
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
TC_LIB_OUT=/tmp/tc_pk0.so TC_NVCC_EXTRA="-DTC_FFMA_PAIRK=0" python paper_1607_00291_b200/_build.py > /dev/null 2>&1 || echo "variant build failed"
timeout 600 python tools/suite.py --no-ttdt --only cfg4_0 > gpurun_out/s_def.jsonl 2>&1
timeout 600 python tools/suite.py --no-ttdt --only cfg4_1 >> gpurun_out/s_def.jsonl 2>&1
TC_B200_LIB=/tmp/tc_pk0.so timeout 600 python tools/suite.py --no-ttdt --only cfg4 > gpurun_out/s_pk0.jsonl 2>&1
TC_KERNEL=ws_nosk timeout 600 python tools/suite.py --no-ttdt --only cfg4 > gpurun_out/s_nosk.jsonl 2>&1
TC_F32_MMA=dmma timeout 600 python tools/suite.py --no-ttdt --only cfg4 > gpurun_out/s_dmma.jsonl 2>&1
python - <<'PY'
import json
def load(p):
    out={}
    for l in open(p):
        try: d=json.loads(l); out[d['config']]=d
        except ValueError: pass
    return out
R=[load('gpurun_out/s_'+x+'.jsonl') for x in ('def','pk0','nosk','dmma')]
print('config                               default   pairk0    no-sk   f32dmma')
for k,d in R[0].items():
    print(f"{k[:34]:34s}", '  '.join(f"{r.get(k,{}).get('vs_gemm',0):7.3f}" for r in R))
PY
