mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "host" 2>&1 | tail -1
TC_HOST_RAMP=0 timeout 600 python tools/e2e_chunks.py 8 12 | sed 's/^/equal /'
timeout 600 python tools/e2e_chunks.py 8 12 | sed 's/^/ramp  /'
