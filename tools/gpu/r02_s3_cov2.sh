# Cluster split-K at the 40% coverage rule (new default) with a per-kernel occupancy cache:
# parity, few-tile sizes with portable (8) and non-portable (16) maxima, then the f2 / f1 /
# baseline suites on the new default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cluster_split or skw or stream_k" 2>&1 | tail -2
SZ=323x323x3000,384x384x4096,512x512x2048,512x512x512,640x640x640,768x768x768,1024x1024x1024
for mx in 8 16; do
  echo "max=$mx"
  TC_CSK_MAX=$mx SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | cut -c1-160
  TC_CSK_DEBUG=1 TC_CSK_MAX=$mx SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | grep "^csk" | sort | uniq
done
timeout 1200 python tools/suite.py --family f2 --no-ttdt > gpurun_out/suite_f2_s3b.jsonl 2>/dev/null
timeout 900 python tools/suite.py --family f1 --no-ttdt > gpurun_out/suite_f1_s3b.jsonl 2>/dev/null
timeout 1500 python tools/suite.py --family baseline --no-ttdt > gpurun_out/suite_base_s3b.jsonl 2>/dev/null
python tools/compare_suites.py profiles/r02/suite_r02s3_f2.jsonl gpurun_out/suite_f2_s3b.jsonl 2>&1 | tail -30
python tools/compare_suites.py profiles/r02/suite_r02s2_f1_final.jsonl gpurun_out/suite_f1_s3b.jsonl 2>&1 | tail -10
python tools/compare_suites.py profiles/r02/suite_r02s3_baseline.jsonl gpurun_out/suite_base_s3b.jsonl 2>&1 | tail -50
