CMD="python tools/suite.py --only cfg4_09_f32 --no-ttdt --reps 2"
timeout 600 $CMD > gpurun_out/plain_f32.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 2 -c 1 -o gpurun_out/prof_f32 $CMD > gpurun_out/ncu_f32.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_f32.log; tail -2 gpurun_out/ncu_f32.log
