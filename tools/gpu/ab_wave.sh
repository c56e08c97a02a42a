# wave alignment A/B on cfg5 (time and DRAM bytes of one launch) and the cfg2/cfg3 suite
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-gemm"
for w in 1 0; do
  TC_WAVE_SYNC=$w timeout 600 $CMD > gpurun_out/wave$w.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/wave$w.log').readlines()[-1]);print('wave_sync=$w', d['value'], d['roofline']['frac'], d['clocks'])"
  TC_WAVE_SYNC=$w timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_ -s 3 -c 1 --csv --log-file gpurun_out/traffic_wave$w.csv $CMD > /dev/null 2>&1
  grep -E "dram__bytes|hit_rate|duration" gpurun_out/traffic_wave$w.csv | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
for w in 1 0; do TC_WAVE_SYNC=$w timeout 600 python tools/suite.py --no-ttdt --only cfg2 > gpurun_out/v_w$w.jsonl 2>&1; TC_WAVE_SYNC=$w timeout 600 python tools/suite.py --no-ttdt --only cfg3 >> gpurun_out/v_w$w.jsonl 2>&1; done
python tools/compare_many.py w1 w0
