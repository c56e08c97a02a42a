# ncu --set full of the fp32/fp64 contraction kernel for one SWEEP_SIZES size (tools/f32_size_sweep.py)
# usage: SWEEP_SIZES=1024x1024x1024 bash tools/gpu/ncu_sweep.sh <name>
n=$1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${NCU_KREGEX:-tc_} -s 3 -c 1 -o gpurun_out/prof_$n python tools/f32_size_sweep.py > gpurun_out/ncu_$n.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_$n.ncu-rep > gpurun_out/summary_$n.txt 2>&1
ncu -i gpurun_out/prof_$n.ncu-rep --page source --csv > gpurun_out/source_$n.csv 2>/dev/null
[ "$KEEP_REP" = "1" ] || rm -f gpurun_out/prof_$n.ncu-rep
