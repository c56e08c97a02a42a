# cfg5 (the bench workload): current build vs the checkpoint-2 build (1a943b6), same box, alternating
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 600 python tools/suite.py --no-ttdt --only cfg5 --reps 3 | sed "s/^/cur /" >> gpurun_out/ck2ab.txt 2>&1
  TC_B200_LIB=build_var/tc_ck2.so timeout 600 python tools/suite.py --no-ttdt --only cfg5 --reps 3 | sed "s/^/ck2 /" >> gpurun_out/ck2ab.txt 2>&1
done
cut -c1-4,100-200 gpurun_out/ck2ab.txt
