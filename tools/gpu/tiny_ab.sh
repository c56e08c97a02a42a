python __graft_entry__.py > gpurun_out/build.log 2>&1
python tools/gpu/tiny_sweep.py > gpurun_out/tiny_default.jsonl 2>&1
for v in "t64n4:-DTC_TINY_THREADS=64 -DTC_TINY_NB=4" "t64n2:-DTC_TINY_THREADS=64 -DTC_TINY_NB=2" "t128n2:-DTC_TINY_THREADS=128 -DTC_TINY_NB=2" "t32n4:-DTC_TINY_THREADS=32 -DTC_TINY_NB=4"; do
  n=${v%%:*}; f=${v#*:}
  TC_LIB_OUT=/tmp/tc_$n.so TC_NVCC_EXTRA="$f" python paper_1607_00291_b200/_build.py > /dev/null 2>&1
  TC_B200_LIB=/tmp/tc_$n.so python tools/gpu/tiny_sweep.py > gpurun_out/tiny_$n.jsonl 2>&1
done
