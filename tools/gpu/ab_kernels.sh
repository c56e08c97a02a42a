# parity of the default kernel, then the small and full bench for each kernel variant
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for K in simple ws; do
  TC_KERNEL=$K timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_$K.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_$K.log').read().strip().splitlines()[-1]);print('$K', d['value'], d['roofline']['frac'], d['same_size_gemm'], d['clocks'])"
done
