# session-2 batch B: HBM write ceilings with 8/16/32-byte per-lane stores vs torch fill_/copy_
mkdir -p gpurun_out
timeout 300 ./build_var/write_bw > gpurun_out/calib_write_bw32.jsonl 2>&1
python - >> gpurun_out/calib_write_bw32.jsonl 2>&1 <<'PY'
import torch, json
x = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
def best(f):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True); f(); torch.cuda.synchronize(); m = 1e9
    for _ in range(10):
        s.record(); f(); e.record(); e.synchronize(); m = min(m, s.elapsed_time(e))
    return m
for name, f, nb in [("torch_fill", lambda: x.fill_(1.0), 8 << 28), ("torch_zero", lambda: x.zero_(), 8 << 28),
                    ("torch_copy", lambda: y.copy_(x), 16 << 28)]:
    print(json.dumps({"kind": name, "gbs": round(nb / best(f) / 1e6)}))
PY
cat gpurun_out/calib_write_bw32.jsonl
