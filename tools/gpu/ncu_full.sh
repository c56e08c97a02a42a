# ncu --set full of the contraction kernel on the half-length cfg5 (same structure), after a clean run
CMD="python bench.py --small --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm"
timeout 600 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 1 -c 1 -o gpurun_out/prof_small $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/plain_small.log; tail -5 gpurun_out/ncu_full.log
