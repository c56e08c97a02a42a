nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/calib_clocks.csv &
SMI=$!
nvidia-smi > gpurun_out/calib_smi.txt
nproc > gpurun_out/calib_host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/calib_host.txt; free -g >> gpurun_out/calib_host.txt
timeout 300 ./tools/calib/bin/fp64_peak > gpurun_out/calib_fp64.jsonl 2>&1
timeout 600 python tools/calib/dgemm_peak.py --big > gpurun_out/calib_dgemm.jsonl 2>&1
kill $SMI
cat gpurun_out/calib_fp64.jsonl gpurun_out/calib_dgemm.jsonl gpurun_out/calib_host.txt
