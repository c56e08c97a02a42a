# parity under both gather policies, then the cfg4 / f1 / f2 suites under each
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
TC_GATHER=mixed timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or random or guard or f32 or loader or strided" 2>&1 | tail -2
for g in elem mixed; do
  TC_GATHER=$g timeout 600 python tools/suite.py --no-ttdt --only cfg4 > gpurun_out/suite_cfg4_$g.jsonl 2>&1
  TC_GATHER=$g timeout 600 python tools/suite.py --no-ttdt --family f2 > gpurun_out/suite_f2_$g.jsonl 2>&1
  TC_GATHER=$g timeout 600 python tools/suite.py --no-ttdt --family f1 > gpurun_out/suite_f1_$g.jsonl 2>&1
done
python tools/compare_suites.py gpurun_out/suite_cfg4_elem.jsonl gpurun_out/suite_cfg4_mixed.jsonl
python tools/compare_suites.py gpurun_out/suite_f2_elem.jsonl gpurun_out/suite_f2_mixed.jsonl
python tools/compare_suites.py gpurun_out/suite_f1_elem.jsonl gpurun_out/suite_f1_mixed.jsonl
