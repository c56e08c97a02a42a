# cluster split-K (TC_CSK, TC_CSK_MAX): parity, then sizes and suites
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster_split or stream_k" 2>&1 | tail -3
for v in "0 8" "1 8" "1 16"; do set -- $v
  echo "csk=$1 max=$2"
  TC_CSK=$1 TC_CSK_MAX=$2 SWEEP_DTYPE=f64 SWEEP_SIZES=256x256x256,512x512x512,768x768x768,1024x1024x1024,1536x1536x1536,256x256x65536 timeout 300 python tools/f32_size_sweep.py | cut -c1-130
  TC_CSK=$1 TC_CSK_MAX=$2 timeout 300 python tools/suite.py --family f2 --no-ttdt --match "f2_1[567]" | cut -c1-200
done
