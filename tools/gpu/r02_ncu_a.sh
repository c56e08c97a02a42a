# Round 2: ncu --set full of the kernels furthest below their rooflines (cfg4 fp64 stragglers,
# cfg4 fp32 on tcgen05, the rank-k and skinny low-intensity kernels).
mkdir -p gpurun_out
FAM=baseline bash tools/gpu/ncu_cases.sh baseline cfg4_11_f64 cfg4_08_f64 cfg4_15_f32 cfg4_05_f32 cfg4_13_f32
FAM=f1 bash tools/gpu/ncu_cases.sh f1 f1_k5 f1_k16
FAM=f2 bash tools/gpu/ncu_cases.sh f2 f2_00 f2_16 f2_05
