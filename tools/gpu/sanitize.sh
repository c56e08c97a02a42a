# one compute-sanitizer tool per call (B200_PROFILING.md); small cases only
TOOL=${1:-memcheck}
SEL="test_cfg1_full_nan_C_beta0 or test_cfg2_ragged or test_stream_k_splits or test_random_small_contractions or test_f32_misaligned_views or test_zero_length or test_strided_subviews or test_f32_loader_directions or test_skinny_shapes or test_negative_strides or test_guard_bands"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" > gpurun_out/plain_sanitize.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" > gpurun_out/sanitize_$TOOL.log 2>&1
echo "sanitize rc=$?" >> gpurun_out/sanitize_$TOOL.log
tail -5 gpurun_out/plain_sanitize.log; tail -15 gpurun_out/sanitize_$TOOL.log
