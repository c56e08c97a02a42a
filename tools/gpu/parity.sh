python __graft_entry__.py smoke > gpurun_out/smoke1.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke1.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not cfg5_full" > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu1.log
tail -5 gpurun_out/smoke1.log; tail -30 gpurun_out/pytest_gpu1.log
