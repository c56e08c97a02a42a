mkdir -p gpurun_out
TC_RANKK_RG=2 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "rankk or f1" 2>&1 | tail -1
for R in 1 2; do for O in 32 64; do TC_RANKK_RG=$R TC_RANKK_OCC2=$O timeout 300 python tools/suite.py --family f1 --only f1_k5 --no-ttdt > /tmp/o.json; python -c "import json; d=json.loads(open('/tmp/o.json').readline()); print('rg=$R occ=$O', d['ms'], d['hbm_gbs'], d['vs_gemm'])"; done; done
