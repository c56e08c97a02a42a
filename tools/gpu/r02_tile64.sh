# fp64 small-tile kernel (tile64.cu): parity forced on every fp64 tile shape, then A/B vs TC_TILE64=0
mkdir -p gpurun_out
TC_TILE64=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_ablation.py -m gpu -q -x -p no:cacheprovider -k "not f32" > gpurun_out/t64_parity_forced.log 2>&1; tail -1 gpurun_out/t64_parity_forced.log
TC_TILE64=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f64 or cfg2 or f2_" > gpurun_out/t64_full_forced.log 2>&1; tail -1 gpurun_out/t64_full_forced.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "f2 or stream_k or sk" > gpurun_out/t64_parity_default.log 2>&1; tail -1 gpurun_out/t64_parity_default.log
for V in 0 D; do
  if [ $V = D ]; then E=""; else E="TC_TILE64=0"; fi
  env $E SWEEP_DTYPE=f64 timeout 600 python tools/f32_size_sweep.py > gpurun_out/t64_sweep_$V.jsonl 2>/dev/null
  env $E timeout 600 python tools/suite.py --family all --no-ttdt --match "f2_1[67]|cfg4_0[08]_f64" > gpurun_out/t64_suite_$V.jsonl 2>/dev/null
done
python - <<'PY'
import json
for kind in ("sweep", "suite"):
    A = [json.loads(l) for l in open(f"gpurun_out/t64_{kind}_0.jsonl")]
    B = [json.loads(l) for l in open(f"gpurun_out/t64_{kind}_D.jsonl")]
    for a, b in zip(A, B):
        name = a.get("config") or "x".join(map(str, a["mnk"]))
        print(f"{name[:34]:34s} ws {a['ms']*1e3:9.1f} us ({a['vs_gemm']:.3f})   tile64-default {b['ms']*1e3:9.1f} us ({b['vs_gemm']:.3f})")
PY
