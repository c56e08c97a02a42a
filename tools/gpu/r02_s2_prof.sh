# per-role barrier-wait cycles of the fp32 tcgen05 kernel (TC_UMMA_PROF build, CTA 0), current build
mkdir -p gpurun_out
for c in ${CASES:-cfg4_04_f32 cfg4_07_f32 cfg4_11_f32 cfg4_12_f32 cfg4_18_f32 cfg4_14_f32 cfg4_02_f32}; do
  echo "== $c" >> gpurun_out/umma_prof2.txt
  TC_B200_LIB=build_var/tc_prof.so timeout 300 python tools/suite.py --no-ttdt --only $c --reps 1 2>&1 | grep -E "PROF" | sort -t' ' -k3 -n | awk '{print $2,$3,$4,$5,$6,$7,$8,$9,$10,$11,$12,$13,$14,$15,$16,$17}' | sort -n -k2 | head -14 >> gpurun_out/umma_prof2.txt
done
cat gpurun_out/umma_prof2.txt
