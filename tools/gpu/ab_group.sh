# DRAM bytes and time of one cfg5 launch for several tile-rasterisation group heights
python __graft_entry__.py > /dev/null 2>&1
for g in 2 4 8 16 32; do
  TC_LIB_OUT=/tmp/tc_g$g.so TC_NVCC_EXTRA="-DTC_GROUP_M=$g" python paper_1607_00291_b200/_build.py > /dev/null 2>&1
  TC_B200_LIB=/tmp/tc_g$g.so timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_ -s 1 -c 1 --csv --log-file gpurun_out/tg_$g.csv python tools/gpu/traffic_probe.py cfg5 > /dev/null 2>&1
  echo "GROUP_M=$g $(grep -E 'dram__bytes|hit_rate|duration' gpurun_out/tg_$g.csv | awk -F'","' '{printf "%s %s  ", $(NF-2), $NF}')"
done
