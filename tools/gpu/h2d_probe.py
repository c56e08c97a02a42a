"""Host<->device copy bandwidth and cudaMallocAsync cost on the box (input to the host-path
pipeline design)."""
import time
import torch

GB = 1 << 30
for size_gb in (1, 4, 12):
    n = size_gb * GB // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{name} {size_gb} GiB pinned: {size_gb * GB / ms / 1e6:.1f} GB/s", flush=True)
    # both directions at once on two streams
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"duplex {size_gb} GiB each way: {2 * size_gb * GB / dt / 1e9:.1f} GB/s total", flush=True)
    del h, d, h2, d2
    torch.cuda.empty_cache()
# pageable
n = 4 * GB // 8
h = torch.empty(n, dtype=torch.float64); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h); torch.cuda.synchronize()
print(f"h2d 4 GiB pageable: {4 * GB / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
import os
print("host cores", len(os.sched_getaffinity(0)))
os.system("nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 'Link Width\\|PCIe Generation' | head -20; free -g")
