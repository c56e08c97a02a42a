# Cluster split-K: 40% coverage and non-portable sizes only for short stream-K pieces (<= 64 K
# steps per CTA). Parity, few-tile sizes, the f2 suite (f2_16 / f2_17 regression check)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cluster_split or skw or stream_k" 2>&1 | tail -2
SZ=323x323x3000,384x384x4096,512x512x2048,512x512x512,640x640x640,768x768x768,1024x1024x1024,256x256x65536
SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | cut -c1-160
TC_CSK_DEBUG=1 SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | grep "^csk" | sort | uniq
timeout 1200 python tools/suite.py --family f2 --no-ttdt > gpurun_out/suite_f2_s3c.jsonl 2>/dev/null
python tools/compare_suites.py profiles/r02/suite_r02s3_f2.jsonl gpurun_out/suite_f2_s3c.jsonl 2>&1 | tail -30
