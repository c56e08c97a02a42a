# per-role barrier-wait cycles of the fp32 tcgen05 kernel (TC_UMMA_PROF build, CTA 0)
mkdir -p gpurun_out
TC_LIB_OUT=/tmp/tc_prof.so TC_NVCC_EXTRA="-DTC_UMMA_PROF" python paper_1607_00291_b200/_build.py > /tmp/b.log 2>&1 || { tail -5 /tmp/b.log; exit 1; }
for c in ${CASES:-cfg4_05_f32 cfg4_15_f32 cfg4_13_f32}; do
 for rp in 1; do
  echo "== $c RP=$rp" >> gpurun_out/umma_prof.txt
  TC_B200_LIB=/tmp/tc_prof.so timeout 300 python tools/suite.py --no-ttdt --only $c --reps 1 2>&1 | grep -E "PROF|gflops" | grep -v "warp 1[345] " | tail -14 >> gpurun_out/umma_prof.txt
 done
done
cat gpurun_out/umma_prof.txt
