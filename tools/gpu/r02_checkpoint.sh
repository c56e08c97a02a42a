# Round-2 checkpoint: smoke, the whole GPU suite, the bench line (N=1) and the reference arm
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/ck_smoke.log 2>&1; tail -3 gpurun_out/ck_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/ck_gputest.log 2>&1; tail -8 gpurun_out/ck_gputest.log
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; cat gpurun_out/ck_bench.json | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/ck_ref.json 2> gpurun_out/ck_ref.err; cut -c1-300 gpurun_out/ck_ref.json
