# Round-2 bench evidence: the bench line, then the launch list of the same command with per-launch
# device time and DRAM bytes (one ncu pass; cold-cache, serialised: compare shares), summarised
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ev_ncu.log 2>&1
echo "ncu rc=$?"
python tools/summarize_launches.py gpurun_out/launches_bench_r02.csv > gpurun_out/launches_bench_r02.summary.txt; cat gpurun_out/launches_bench_r02.summary.txt
cut -c1-300 gpurun_out/ev_bench.json
