# ncu captures of the fig:bench stragglers f2_05 / f2_15 / f2_16 at full size
mkdir -p gpurun_out
for c in f2_05 f2_15 f2_16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ -c 1 -o gpurun_out/$c -f \
    python tools/suite.py --family f2 --no-ttdt --match "$c" > gpurun_out/ncu_$c.log 2>&1
  echo $c $?
done
