# quick check: stream-K / weighted / cluster split-K parity, then the bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "stream_k or weights or csk or cluster or split" > gpurun_out/q_tests.log 2>&1; tail -2 gpurun_out/q_tests.log
timeout 900 python bench.py > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; cut -c1-240 gpurun_out/q_bench.json
