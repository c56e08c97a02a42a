timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python tools/suite.py --no-ttdt > gpurun_out/suite_sk.jsonl 2> gpurun_out/suite_sk.err; tail -2 gpurun_out/suite_sk.err
TC_KERNEL=ws_nosk timeout 600 python tools/suite.py --no-ttdt --only cfg2 > gpurun_out/suite_nosk.jsonl 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_sk.log 2>&1; tail -1 gpurun_out/bench_sk.log | cut -c1-300
