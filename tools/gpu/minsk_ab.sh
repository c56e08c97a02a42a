# stream-K minimum iterations per CTA (TC_MIN_SK_ITERS) on medium GEMM sizes, fp64 and fp32
python __graft_entry__.py > gpurun_out/build.log 2>&1
export SWEEP_SIZES=512x512x512,768x768x768,1024x1024x1024,1536x1536x1536
for v in 8 4 16 32; do
  TC_LIB_OUT=/tmp/tc_ms$v.so TC_NVCC_EXTRA="-DTC_MIN_SK_ITERS=$v" python paper_1607_00291_b200/_build.py > /dev/null 2>&1
  SWEEP_DTYPE=f64 TC_B200_LIB=/tmp/tc_ms$v.so python tools/f32_size_sweep.py > gpurun_out/ms64_$v.jsonl 2>&1
  TC_B200_LIB=/tmp/tc_ms$v.so python tools/f32_size_sweep.py > gpurun_out/ms32_$v.jsonl 2>&1
done
