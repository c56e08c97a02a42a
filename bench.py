"""Benchmark: fp64 tensor-contraction GFLOP/s (BASELINE.json `metric`) on 1/2/4/8 B200s.

Workload (BASELINE.json configs[4], the 1/2/4/8-GPU config; fits one GPU): cfg5
  C_abcijk = A_abdilm * B_dclmjk, a,b,c,d = 48, i,j,k,l,m = 24, N(0,1) inputs, alpha=1, beta=0
  M x N x K = 55296 x 27648 x 27648 (8.45e13 flops per step), 30.6 GB of operands (>> 126 MB L2).
A step is one full contraction pass (all §8(a) rows: plan lookup, staging, DMMA, epilogue).
With N GPUs, C is sharded over free blocks of (a, b, c) after one NCCL
distribution of A and B from rank 0 (each rank receives the slabs its block reads,
paper_1607_00291_b200/dist.py); K is never split, so there is no data-path
collective. Total work is fixed as N grows -> "scaling": "strong".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--small]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints one JSON line on rank 0. `value` is device-timed (CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks) with inputs resident in HBM; `e2e` is the
same metric through tc_contract_host (host buffers, H2D + D2H inside the timed region).
`--impl reference` times the oracle (oracle/contract.c) on host cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

SHARD_LABELS = "abc"
PEAKS_FILE = os.path.join(ROOT, "profiles", "PEAKS_FP64.json")
# DRAM bytes per launch of the contraction kernel on the full cfg5 workload, from
# `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` of this same
# command (tools/gpu/r02_s2_ck6.sh, the launch list of the final round-2 build); the counters of
# the `--set full` memory section.
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02", "launches_bench_r02s2.csv")


def ncu_traffic(path, kernel_prefix="tc_dmma_ws_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum of the first profiled launch of the kernel."""
    import csv
    if not os.path.exists(path):
        return None
    vals = {}
    for r in csv.reader(open(path)):
        if len(r) < 15 or r[0] == "ID" or kernel_prefix not in r[4]:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(r[13])
        if scale and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            vals.setdefault(r[12], float(r[14].replace(",", "")) * scale)
    if len(vals) != 2:
        return None
    return int(sum(vals.values()))
SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--small", action="store_true", help="cfg5 at half lengths (quick check)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gemm", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--distribute", default="slabs", choices=["slabs", "broadcast"],
                    help="N>1 operand distribution: per-rank slabs (send/recv) or full broadcast")
    return ap.parse_args()


def workload(small: bool):
    return W.cfg5(24, 12) if small else W.cfg5()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------------------------

class Clocks:
    def __init__(self, gpus):
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
        self.gpus = gpus
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((int(f[1]), int(f[2]), float(f[3]), f[5], f[6], f[7], f[8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r[2] > 300] or rows
        reasons = set()
        for r in rows:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in loaded),
                "sm_max_mhz": max(r[1] for r in rows), "power_w_max": max(r[2] for r in rows),
                "samples": len(rows), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------------------------
# oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------------

def oracle_sample(case, A, B, C, target_s=12.0, max_threads=None):
    """Time the oracle on a sampled sub-block of the workload (some indices of every free label,
    all of every bound label) so one run costs ~target_s seconds. Returns (GFLOP/s, cores,
    description)."""
    import oracle
    threads = max_threads or len(os.sched_getaffinity(0))
    rs = np.random.RandomState(0)

    def make(per):
        sel = {x: torch.tensor(sorted(rs.choice(case.lens[x], size=min(per[x], case.lens[x]),
                                                replace=False).tolist()))
               for x in case.lab_c}

        def sub(T, labels):
            for d, x in enumerate(labels):
                if x in sel:
                    T = T.index_select(d, sel[x].to(T.device))
            return T.cpu().contiguous()
        return sel, sub(A, case.lab_a), sub(B, case.lab_b), sub(C, case.lab_c)

    per = {x: 2 for x in case.lab_c}
    for _ in range(6):   # grow the sample evenly over the free labels until ~target_s
        sel, a, b, c = make(per)
        cc = c.clone()
        t0 = time.perf_counter()
        oracle.contract(case.spec, a, b, cc, case.alpha, case.beta, threads=threads)
        dt = time.perf_counter() - t0
        if dt >= 0.5 * target_s or all(per[x] >= case.lens[x] for x in per):
            break
        grow = min(2.0, (target_s / max(dt, 1e-4)) ** (1.0 / len(per)))
        per = {x: max(2, min(case.lens[x], int(round(per[x] * grow)))) for x in per}
    free = math.prod(len(v) for v in sel.values())
    kbound = math.prod(case.lens[x] for x in case.lab_a if x not in case.lab_c)
    flops = 2.0 * free * kbound
    desc = (f"{free} of {math.prod(case.lens[x] for x in case.lab_c)} C elements "
            f"({'x'.join(str(len(sel[x])) for x in case.lab_c)} indices of {case.lab_c}), "
            f"each a full {kbound}-term sum; {flops / 1e9:.1f} GFLOP in {dt:.1f} s")
    return flops / dt / 1e9, threads, desc, (sel, a, b, c, flops)


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle
    case = workload(args.small)
    threads = len(os.sched_getaffinity(0))
    # inputs: generated on the host (the oracle reads host memory only); bounded sample
    gen_dev = "cuda" if torch.cuda.is_available() else "cpu"
    A, B, C = W.make_tensors(case, gen_dev)
    _, _, desc, (sel, a, b, c, flops) = oracle_sample(case, A, B, C, target_s=8.0)
    del A, B, C
    times = []
    for it in range(args.warmup + args.steps):
        cc = c.clone()
        t0 = time.perf_counter()
        oracle.contract(case.spec, a, b, cc, case.alpha, case.beta, threads=threads)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    t = max(times)  # slowest step, like max over ranks; the sample is the same every step
    value = flops / (sum(times) / len(times)) / 1e9
    line = {
        "metric": "fp64 contraction GFLOP/s", "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": case.name, "spec": case.spec, "lens": case.lens,
                   "sample": desc},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": threads,
                         "kind": "oracle", "sample": desc},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------------------------

def timed_loop(fn, steps, stream, world):
    """Barrier + synchronize, CUDA events on `stream` around `steps` calls, barrier + sync;
    returns (max over ranks of the elapsed ms, per-call ms list on this rank)."""
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    total = ev[0].elapsed_time(ev[-1])
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return total, per


def distribution_bytes(case, world, scheme):
    """Modelled bytes of the operand distribution: what rank 0 sends and what each other rank
    receives (dist.plan_traffic; a ring broadcast sends each byte out of its root once)."""
    from paper_1607_00291_b200 import dist as tdist
    ops = [(case.lab_a, 8), (case.lab_b, 8)]
    if scheme == "broadcast":
        full = sum(8 * math.prod(case.shape(lab)) for lab, _ in ops)
        return {"scheme": "broadcast", "src_egress": full, "recv_per_rank": full}
    m = tdist.plan_traffic(world, case.lens, SHARD_LABELS, ops)
    return {"scheme": "slabs (send to slab-group leader + group broadcast)",
            "src_egress": m["src_egress"], "recv_per_rank": max(m["recv"])}


def run_native(args):
    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1607_00291_b200 as tc
    from paper_1607_00291_b200 import dist as tdist

    case = workload(args.small)
    spec, lens = case.spec, case.lens
    stream = torch.cuda.current_stream()

    # -- inputs: seeded on rank 0's GPU and distributed once over NCCL (the one exchange step):
    # by default each rank receives only the A and B slabs its block of C reads (dist.distribute:
    # rank 0 sends each distinct slab once to its group's leader, which broadcasts it within the
    # group); --distribute broadcast sends everyone the full operands instead
    t_b0 = time.perf_counter()
    slabs = world > 1 and args.distribute == "slabs"
    A = B = None
    if rank == 0:
        A, B, c_full = W.make_tensors(case, "cuda")
        del c_full   # the timed C is this rank's shard, allocated below
        torch.cuda.empty_cache()
    elif not slabs:
        A = W.colmajor_view(torch.empty(math.prod(case.shape(case.lab_a)), dtype=torch.float64,
                                        device="cuda"), case.shape(case.lab_a))
        B = W.colmajor_view(torch.empty(math.prod(case.shape(case.lab_b)), dtype=torch.float64,
                                        device="cuda"), case.shape(case.lab_b))
    bcast_ms = None
    recv_elems = None
    ranges = tdist.shard_ranges(world, rank, lens, SHARD_LABELS) if world > 1 else {}
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if slabs:
            As, Bs, recv_elems, _ = tdist.distribute_slabs(spec, A, B, lens, SHARD_LABELS, world,
                                                           rank, dtype=torch.float64, device="cuda")
            A = B = None   # rank 0 keeps dense copies of its own slabs, like every other rank
        else:
            flatA = torch.as_strided(A, (A.numel(),), (1,))
            flatB = torch.as_strided(B, (B.numel(),), (1,))
            tdist.broadcast_operands([flatA, flatB], 0)
        e1.record()
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
        t = torch.tensor([bcast_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)     # the distribution ends on its slowest rank
        bcast_ms = float(t.item())
        torch.cuda.empty_cache()
    cshape = tdist.shard_shape(case.lab_c, lens, ranges)
    C = W.colmajor_view(torch.full((math.prod(cshape),), float("nan"), dtype=torch.float64,
                                   device="cuda"), cshape)
    if not slabs:
        As = tdist.narrow(A, case.lab_a, ranges)
        Bs = tdist.narrow(B, case.lab_b, ranges)
    flops_rank = tdist.shard_flops(spec, lens, ranges)
    flops_total = case.flops()
    plan = tc.Plan.for_tensors(spec, As, Bs, C)
    info = plan.info()

    def step():
        tc.contract(spec, As, Bs, C, case.alpha, case.beta, stream=stream)

    for _ in range(args.warmup):
        step()
    clocks = Clocks(list(range(world)) if world > 1 else [local])
    if rank == 0:
        clocks.start()
    total_ms, per = timed_loop(step, args.steps, stream, world)
    clk = clocks.stop() if rank == 0 else None
    ms_step = total_ms / args.steps
    value = flops_total / (ms_step * 1e-3) / 1e9             # GFLOP/s, whole job
    kernel_ms = statistics.mean(per)                         # one kernel launch per step
    achieved_tf = flops_rank / (kernel_ms * 1e-3) / 1e12
    torch.cuda.synchronize()
    finite = bool(torch.isfinite(C).all().item())

    # -- same-size GEMM (cuBLAS DGEMM, equal M, N, K of this rank's shard)
    gemm_tf = None
    if not args.no_gemm:
        m, n, k = info["m"], info["n"], info["k"]
        del_list = []
        try:
            Ga = torch.randn(m, k, dtype=torch.float64, device="cuda")
            Gb = torch.randn(k, n, dtype=torch.float64, device="cuda")
            Gc = torch.empty(m, n, dtype=torch.float64, device="cuda")
            del_list = [Ga, Gb, Gc]
            torch.mm(Ga, Gb, out=Gc)
            gsteps = max(1, min(args.steps, 3))
            gms, _ = timed_loop(lambda: torch.mm(Ga, Gb, out=Gc), gsteps, stream, world)
            gemm_tf = 2.0 * m * n * k / (gms / gsteps * 1e-3) / 1e12
        except torch.OutOfMemoryError:
            gemm_tf = None
        del del_list
        torch.cuda.empty_cache()

    # -- end to end through tc_contract_host: host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        hA = W.colmajor_view(torch.empty(As.numel(), dtype=torch.float64, pin_memory=True),
                             list(As.shape))
        hB = W.colmajor_view(torch.empty(Bs.numel(), dtype=torch.float64, pin_memory=True),
                             list(Bs.shape))
        hC = W.colmajor_view(torch.empty(C.numel(), dtype=torch.float64, pin_memory=True),
                             list(C.shape))
        hA.copy_(As)
        hB.copy_(Bs)
        del A, B
        As = Bs = None
        torch.cuda.empty_cache()

        def estep():
            tc.contract_host(spec, hA, hB, hC, case.alpha, case.beta, stream=stream)

        estep()
        esteps = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(esteps):
            estep()
        e1.record(stream)
        torch.cuda.synchronize()
        el = e0.elapsed_time(e1) * 1e-3
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        # at N > 1 each rank's inputs are its own slabs in host memory (one node: every GPU
        # copies over its own PCIe link); the device-side distribution of the resident-input
        # run is reported beside it as if it were paid once per step (value_incl_distribution)
        e2e = {"value": round(flops_total / (el / esteps) / 1e9, 2), "unit": "GFLOP/s",
               "value_incl_distribution": None if bcast_ms is None else round(
                   flops_total / (el / esteps + bcast_ms * 1e-3) / 1e9, 2),
               "h2d_bytes_per_step": (hA.numel() + hB.numel()) * 8 * world,
               "d2h_bytes_per_step": hC.numel() * 8 * world,
               "steps": esteps, "ms_per_step": round(1e3 * el / esteps, 2),
               "timer": "CUDA events around synchronous tc_contract_host calls, max over ranks"}

    # -- cpu baseline: the oracle on a bounded sample (rank 0 at N=1 only)
    cpu = None
    if not args.no_cpu and world == 1:
        if As is None:
            A_ref, B_ref = hA, hB
        else:
            A_ref, B_ref = As, Bs
        v, cores, desc, _ = oracle_sample(case, A_ref, B_ref, C, target_s=12.0)
        cpu = {"value": round(v, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
               "sample": desc}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    peak = peaks.get("dmma_tflops", 37.13)
    line = {
        "metric": "fp64 contraction GFLOP/s", "value": round(value, 2), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": case.name, "spec": spec, "lens": lens,
                   "mnk": [info["m"], info["n"], info["k"]], "flops_per_step": flops_total,
                   "parallelism": ("1 GPU, whole contraction" if world == 1 else
                                   f"shard C over ({SHARD_LABELS}) x{world}, " + (
                                       "NCCL send/recv of per-rank A,B slabs" if slabs
                                       else "NCCL broadcast of A,B")),
                   "shard_ranges_rank0": ranges, "l2": "inputs larger than L2 (30.6 GB >> 126 MB)",
                   "distribute": args.distribute if world > 1 else None,
                   "distribute_ms": bcast_ms, "received_elems_rank": recv_elems,
                   "distribution_bytes": None if world == 1 else distribution_bytes(
                       case, world, args.distribute),
                   "plan": info},
        "pct_fp64_peak": round(100 * value / 1e3 / (peak * world), 2),
        "same_size_gemm": None if gemm_tf is None else {
            "kind": "cuBLAS DGEMM (torch.mm float64) of the rank-0 shard's M x N x K",
            "tflops_per_gpu": round(gemm_tf, 2),
            "contraction_over_gemm": round(achieved_tf / gemm_tf, 4)},
        "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3),
                     "peak": peak, "unit": "TFLOP/s", "frac": round(achieved_tf / peak, 4),
                     "traffic": None if args.small or world > 1 else ncu_traffic(TRAFFIC_FILE),
                     "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, one "
                                       "launch of this workload (profiles/r02/launches_bench_r02s2.csv)",
                     "peak_source": "profiles/PEAKS_FP64.json dmma_tflops (measured DMMA.8x8x4 "
                                    "loop on this pool's B200; fp64 has no entry in "
                                    "MEASURED_PEAKS.json)",
                     "kernel": "tc_dmma_ws_kernel (persistent, warp-specialised DMMA)", "kernel_ms": round(kernel_ms, 3),
                     "algorithmic_flops_per_launch": flops_rank},
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": args.steps * world,
        "finite_output": finite,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
