mkdir -p gpurun_out
timeout 300 ./build_var/write_bw > gpurun_out/calib_write_bw32b.jsonl 2>&1
grep chunk gpurun_out/calib_write_bw32b.jsonl
