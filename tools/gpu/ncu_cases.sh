# ncu --set full of the contraction kernel for each named suite case (after a clean run of each);
# writes text summaries (tools/ncu_summary.py) and drops the .ncu-rep unless KEEP_REP=1
# usage: bash tools/gpu/ncu_cases.sh <family> <case-prefix> [<case-prefix> ...]
fam=$1; shift
for c in "$@"; do
  CMD="python tools/suite.py --family ${FAM:-baseline} --only $c --no-ttdt --reps 2"
  timeout 600 $CMD > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KREGEX:-tc_} -s 2 -c 1 -o gpurun_out/prof_$c $CMD > gpurun_out/ncu_$c.log 2>&1
  echo "$c ncu rc=$?"; head -1 gpurun_out/plain_$c.log
  python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/summary_$c.txt 2>&1
  ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv > gpurun_out/source_$c.csv 2>/dev/null
  [ "$KEEP_REP" = "1" ] || rm -f gpurun_out/prof_$c.ncu-rep
done
