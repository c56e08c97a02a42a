# cfg5: bench value and one launch's DRAM traffic per tile-rasterisation group height (TC_GROUP_M)
python __graft_entry__.py > gpurun_out/build.log 2>&1
for g in "$@"; do
  TC_LIB_OUT=/tmp/tc_g$g.so TC_NVCC_EXTRA="-DTC_GROUP_M=$g" python paper_1607_00291_b200/_build.py > /dev/null 2>&1 || echo "build $g failed"
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-gemm"
  TC_B200_LIB=/tmp/tc_g$g.so timeout 600 $CMD > gpurun_out/bench_g$g.json 2>/dev/null
  TC_B200_LIB=/tmp/tc_g$g.so timeout 900 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:tc_ -s 3 -c 1 --csv --log-file gpurun_out/traffic_g$g.csv $CMD > /dev/null 2>&1
  echo "GROUP_M=$g $(python -c "import json;d=json.load(open('gpurun_out/bench_g$g.json'));print(d['value'], d['clocks'])") $(grep -o '"dram__bytes_read.sum","byte","[0-9]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.]*"' gpurun_out/traffic_g$g.csv | tr '\n' ' ')"
done
