# stream-K pieces per tile cap (TC_MAX_PIECES) on few-tile long-K shapes, fp64 and fp32
python __graft_entry__.py > gpurun_out/build.log 2>&1
export SWEEP_SIZES=256x256x65536,512x512x16384,128x128x262144
for v in 16 32 48; do
  TC_LIB_OUT=/tmp/tc_mp$v.so TC_NVCC_EXTRA="-DTC_MAX_PIECES=$v" python paper_1607_00291_b200/_build.py > /dev/null 2>&1
  SWEEP_DTYPE=f64 TC_B200_LIB=/tmp/tc_mp$v.so python tools/f32_size_sweep.py > gpurun_out/mp64_$v.jsonl 2>&1
  TC_B200_LIB=/tmp/tc_mp$v.so python tools/f32_size_sweep.py > gpurun_out/mp32_$v.jsonl 2>&1
done
