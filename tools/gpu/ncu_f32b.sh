for C in cfg4_08_f32 cfg4_16_f32; do
CMD="python tools/suite.py --only $C --no-ttdt --reps 2"
timeout 600 $CMD > gpurun_out/plain_$C.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 2 -c 1 -o gpurun_out/prof_$C $CMD > gpurun_out/ncu_$C.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$C.log; tail -1 gpurun_out/ncu_$C.log
done
