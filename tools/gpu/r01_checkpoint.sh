# Round-1 checkpoint: build check, smoke, GPU parity suite, default bench line, launch list,
# DRAM traffic of one full-size contraction launch, ncu --set full of the half-length cfg5.
set -x
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo "build rc=$?" >> gpurun_out/build.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-gemm"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_ -s 3 -c 1 --csv --log-file gpurun_out/traffic_full.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?" >> gpurun_out/ncu_traffic.log
CMDS="python bench.py --small --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm"
timeout 600 $CMDS > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 1 -c 1 -o gpurun_out/prof_small $CMDS > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/build.log; tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.log; tail -5 gpurun_out/bench.err; for f in gpurun_out/ncu_launch.log gpurun_out/ncu_traffic.log gpurun_out/ncu_full.log; do tail -n 3 $f; done
python tools/ncu_summary.py gpurun_out/prof_small.ncu-rep > gpurun_out/summary_small.txt 2>&1; ncu -i gpurun_out/prof_small.ncu-rep --page source --csv > gpurun_out/source_small.csv 2>/dev/null; rm -f gpurun_out/prof_small.ncu-rep
