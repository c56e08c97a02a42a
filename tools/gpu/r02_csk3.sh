timeout 900 python -m pytest tests -m gpu -x -q -k "cluster_split" 2>&1 | tail -2
for v in "0 8" "1 8" "1 16"; do set -- $v
  echo "csk=$1 max=$2"
  TC_CSK_DEBUG=1 TC_CSK=$1 TC_CSK_MAX=$2 SWEEP_DTYPE=f64 SWEEP_SIZES=512x512x512,640x640x640,768x768x768,384x384x4096,256x256x65536 timeout 300 python tools/f32_size_sweep.py 2>&1 | grep -v "^csk" | cut -c1-130
done
TC_CSK_DEBUG=1 SWEEP_DTYPE=f64 SWEEP_SIZES=512x512x512 timeout 300 python tools/f32_size_sweep.py 2>&1 | grep "^csk" | head -2
