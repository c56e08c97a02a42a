# session-2 batch A: warp-map A/B on cfg5 + cfg4 fp64 (same box, alternating), fresh ncu of
# slow cfg4 fp32 cases on the current build
mkdir -p gpurun_out
for rep in 1 2; do
  for v in default oldmap; do
    lib=""; [ $v = oldmap ] && lib=build_var/tc_oldmap.so
    TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --only cfg5 --reps 3 >> gpurun_out/map_$v.jsonl 2>&1
    TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --only cfg4_1 --reps 5 >> gpurun_out/map_$v.jsonl 2>&1
  done
done
bash tools/gpu/ncu_cases.sh baseline cfg4_08_f32 cfg4_18_f32 cfg4_14_f32
