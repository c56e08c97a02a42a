# Round-2 session-3 checkpoint 10 (cluster split-K sizes / coverage): smoke, whole GPU suite,
# bench (N=1), reference arm, bench launch list
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/ck10_smoke.log 2>&1; tail -3 gpurun_out/ck10_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/ck10_gputest.log 2>&1; tail -4 gpurun_out/ck10_gputest.log
timeout 900 python bench.py > gpurun_out/ck10_bench.json 2> gpurun_out/ck10_bench.err; cut -c1-300 gpurun_out/ck10_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/ck10_ref.json 2> gpurun_out/ck10_ref.err; cut -c1-200 gpurun_out/ck10_ref.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench_r02s3.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ck10_ncu.log 2>&1
echo "ncu rc=$?"
python tools/summarize_launches.py gpurun_out/launches_bench_r02s3.csv > gpurun_out/launches_bench_r02s3.summary.txt; head -12 gpurun_out/launches_bench_r02s3.summary.txt
