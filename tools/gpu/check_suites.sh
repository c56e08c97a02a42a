# build, full GPU parity, then the given suite families (default: baseline f1 f2)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf 2>&1 | grep -E "^FAILED|passed|failed"
for fam in ${@:-baseline f1 f2}; do
  timeout 900 python tools/suite.py --no-ttdt --family $fam > gpurun_out/suite_$fam.jsonl 2>gpurun_out/suite_$fam.err
  python tools/compare_suites.py gpurun_out/suite_$fam.jsonl gpurun_out/prev_suite_$fam.jsonl 2>/dev/null || cat gpurun_out/suite_$fam.jsonl
done
