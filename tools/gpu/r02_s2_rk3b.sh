# rank-k v3 CTA-tile forms (exact-K instantiations): parity, then f1 k5 A/B against v2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "rankk" > gpurun_out/rk3_tests.log 2>&1; tail -2 gpurun_out/rk3_tests.log
for rep in 1 2; do
  for f in 0 1 2 3; do
    TC_RANKK3_FORM=$f timeout 600 python tools/suite.py --no-ttdt --family f1 --only f1_k5_ --reps 10 | sed "s/^/form$f /" >> gpurun_out/rk3b.txt 2>&1
  done
  TC_RANKK_V=2 timeout 600 python tools/suite.py --no-ttdt --family f1 --only f1_k5_ --reps 10 | sed "s/^/v2 /" >> gpurun_out/rk3b.txt 2>&1
done
cut -c1-40,150-260 gpurun_out/rk3b.txt
