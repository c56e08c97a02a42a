# Cluster split-K with cluster sizes 5-7 (not only 8 and 4): parity, then graph-timed fp64 sizes
# against the power-of-two policy (TC_CSK_POW2=1) and cuBLAS
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cluster_split" 2>&1 | tail -2
SZ=512x512x512,640x640x640,512x640x768,576x576x576,768x768x768,500x380x900,384x384x4096,1024x1024x1024
for rep in 1 2; do
for p in 1 0; do
  echo "pow2=$p"
  TC_CSK_POW2=$p SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | cut -c1-160
done
done
TC_CSK_DEBUG=1 SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | grep "^csk" | sort | uniq
