# fp64 few-tile regime: stream-K piece length (TC_WS_MINSK) and no split (TC_KERNEL=ws_nosk)
for v in 4 8 16 32 1000; do
  echo "minsk=$v"; TC_WS_MINSK=$v SWEEP_DTYPE=f64 SWEEP_SIZES=256x256x256,512x512x512,768x768x768 timeout 300 python tools/f32_size_sweep.py | cut -c1-120
done
echo nosk; TC_KERNEL=ws_nosk SWEEP_DTYPE=f64 SWEEP_SIZES=256x256x256,512x512x512,768x768x768 timeout 300 python tools/f32_size_sweep.py | cut -c1-120
