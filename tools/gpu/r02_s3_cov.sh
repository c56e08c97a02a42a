# Cluster split-K coverage rule (T S >= cov% of stream-K's CTAs; default 80) with sizes up to 16,
# on few-tile long-K fp64 shapes that stream-K serves today; then f2_09 / f2_16 with and without
# the 5-7 sizes (noise check of the suite run)
mkdir -p gpurun_out
SZ=323x323x3000,384x384x4096,768x768x768,256x256x65536,512x512x2048,640x384x6000
for v in "80 8" "60 8" "40 8" "60 16" "40 16"; do set -- $v
  echo "cov=$1 max=$2"
  TC_CSK_COV=$1 TC_CSK_MAX=$2 SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | cut -c1-160
  TC_CSK_DEBUG=1 TC_CSK_COV=$1 TC_CSK_MAX=$2 SWEEP_DTYPE=f64 SWEEP_SIZES=$SZ timeout 300 python tools/f32_size_sweep.py 2>&1 | grep "^csk" | sort | uniq
done
for p in 1 0 1 0; do
  echo "pow2=$p"
  TC_CSK_POW2=$p timeout 300 python tools/suite.py --family f2 --match 'f2_(08|09|16)' --no-ttdt --reps 20 2>/dev/null | cut -c1-200
done
