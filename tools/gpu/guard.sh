timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
timeout 900 python tools/suite.py --only cfg4 --no-ttdt > gpurun_out/suite_cfg4.jsonl 2> gpurun_out/suite_cfg4.err; tail -2 gpurun_out/suite_cfg4.err
