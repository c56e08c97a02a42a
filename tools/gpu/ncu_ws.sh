CMD="python bench.py --small --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm"
export TC_KERNEL=${TC_KERNEL:-ws}
timeout 600 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 1 -c 1 -o gpurun_out/prof_ws $CMD > gpurun_out/ncu_ws.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_ws.log; tail -2 gpurun_out/ncu_ws.log
