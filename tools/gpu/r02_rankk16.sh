mkdir -p gpurun_out
TC_RANKK16=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "rankk or f1" > gpurun_out/rk16_parity.log 2>&1; tail -1 gpurun_out/rk16_parity.log
for c in f1_k5 f1_k16; do for R in 0 1; do TC_RANKK16=$R timeout 300 python tools/suite.py --family f1 --only $c --no-ttdt > /tmp/o.json; python -c "import json; d=json.loads(open('/tmp/o.json').readline()); print('$c rankk16=$R', d['ms'], d['hbm_gbs'], d['vs_gemm'])"; done; done
