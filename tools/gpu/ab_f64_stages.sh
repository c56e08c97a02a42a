# fp64 ring depth A/B on the bench workload (cfg5) and the fp64 suite cases
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for v in 5 6; do TC_LIB_OUT=/tmp/tc_d$v.so TC_NVCC_EXTRA="-DTC_STAGES_F64=$v" python paper_1607_00291_b200/_build.py > /dev/null 2>&1; done
for v in def 5 6; do
  lib=""; [ $v != def ] && lib=/tmp/tc_d$v.so
  TC_B200_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-gemm > gpurun_out/b_d$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b_d$v.log').readlines()[-1]); print('stages=$v', d['value'], d['roofline']['frac'])"
  TC_B200_LIB=$lib timeout 600 python tools/suite.py --no-ttdt --only cfg > gpurun_out/v_d$v.jsonl 2>&1
done
python tools/compare_many.py ddef d5 d6 | grep -v f32
