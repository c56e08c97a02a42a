# ncu of the fp32 tcgen05 kernel after the round-2 gather changes, plus per-role barrier waits
mkdir -p gpurun_out
FAM=baseline bash tools/gpu/ncu_cases.sh baseline cfg4_13_f32 cfg4_15_f32 cfg4_05_f32
rm -f gpurun_out/umma_prof.txt
CASES="cfg4_05_f32 cfg4_15_f32 cfg4_13_f32" bash tools/gpu/r02_umma_prof.sh > /dev/null 2>&1
grep -E "==|warp (0|4|8|12) |gflops" gpurun_out/umma_prof.txt | cut -c1-150
