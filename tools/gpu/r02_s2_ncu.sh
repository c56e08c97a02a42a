# final-build ncu --set full captures: the bench kernel on half-length cfg5, and the fp32 tcgen05
# kernel on cfg4_07 (gather modes 8 + 12) and cfg4_13; text summaries only
mkdir -p gpurun_out
CMD="python bench.py --small --steps 1 --warmup 1 --no-e2e --no-cpu --no-gemm"
timeout 600 $CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_dmma -s 1 -c 1 -o gpurun_out/prof_small $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_small.ncu-rep > gpurun_out/summary_cfg5small_final.txt 2>&1
rm -f gpurun_out/prof_small.ncu-rep
bash tools/gpu/ncu_cases.sh baseline cfg4_07_f32 cfg4_13_f32
