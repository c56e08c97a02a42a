# Round 2: per-config suites with the TTDT comparator (time + workspace bytes) and the SMTC
# ablation (TC_FORCE_PATH=scatter, read per call) on the current kernels.
mkdir -p gpurun_out
timeout 1500 python tools/suite.py --smtc --family baseline > gpurun_out/suite_r02_baseline.jsonl 2> gpurun_out/suite_r02_baseline.err
timeout 600 python tools/suite.py --smtc --family f1 > gpurun_out/suite_r02_f1.jsonl 2> gpurun_out/suite_r02_f1.err
timeout 900 python tools/suite.py --smtc --family f2 > gpurun_out/suite_r02_f2.jsonl 2> gpurun_out/suite_r02_f2.err
wc -l gpurun_out/suite_r02_*.jsonl; for f in gpurun_out/suite_r02_*.err; do tail -n 3 "$f"; done
