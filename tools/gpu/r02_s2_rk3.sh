# rank-k v3 (one-shot grid of 256 x 8 tiles): parity, then f1 A/B against v2 (same box)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "rankk" > gpurun_out/rk3_tests.log 2>&1; tail -3 gpurun_out/rk3_tests.log
for rep in 1 2; do
  timeout 600 python tools/suite.py --no-ttdt --family f1 --only f1_k5 --reps 10 >> gpurun_out/rk3_v3.jsonl 2>&1
  TC_RANKK_V=2 timeout 600 python tools/suite.py --no-ttdt --family f1 --only f1_k5 --reps 10 >> gpurun_out/rk3_v2.jsonl 2>&1
done
timeout 600 python tools/suite.py --no-ttdt --family f1 --reps 5 > gpurun_out/rk3_f1_all.jsonl 2>&1
cat gpurun_out/rk3_v3.jsonl gpurun_out/rk3_v2.jsonl | cut -c1-260
cut -c1-200 gpurun_out/rk3_f1_all.jsonl
