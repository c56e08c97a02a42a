timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python tools/suite.py --family f2 > gpurun_out/suite_f2.jsonl 2> gpurun_out/suite_f2.err; tail -2 gpurun_out/suite_f2.err
timeout 900 python tools/suite.py --family f1 > gpurun_out/suite_f1.jsonl 2> gpurun_out/suite_f1.err; tail -2 gpurun_out/suite_f1.err
TC_FORCE_PATH=scatter timeout 900 python tools/suite.py --family f2 --no-ttdt > gpurun_out/suite_f2_smtc.jsonl 2>&1
TC_FORCE_PATH=scatter timeout 900 python tools/suite.py --no-ttdt --only cfg > gpurun_out/suite_base_smtc.jsonl 2>&1
