# Round-2 session-3 checkpoint 9 (HEAD after the skinny L2-hint switch): smoke, whole GPU suite,
# bench (N=1), reference arm
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/ck9_smoke.log 2>&1; tail -3 gpurun_out/ck9_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/ck9_gputest.log 2>&1; tail -4 gpurun_out/ck9_gputest.log
timeout 900 python bench.py > gpurun_out/ck9_bench.json 2> gpurun_out/ck9_bench.err; cut -c1-300 gpurun_out/ck9_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/ck9_ref.json 2> gpurun_out/ck9_ref.err; cut -c1-200 gpurun_out/ck9_ref.json
