"""One-GPU measurement of the multi-GPU shards of cfg5 (the bench workload): for N = 1, 2, 4, 8 the
rank-0 block of C (dist.shard_ranges over free labels a, b, c) is contracted through the
same C-ABI call the N-GPU bench makes per rank, timed with CUDA events, next to cuBLAS DGEMM of the
shard's M x N x K. Also prints the modelled operand distribution (dist.plan_traffic) and its time
at the measured NVLink peer bandwidth (770 GB/s per direction, B200_PROFILING.md). This is a
projection, not a multi-GPU measurement: ranks share nothing at run time except the one-off
distribution, so the per-shard time on one GPU is what each GPU of an N-GPU run computes.

    python tools/shard_bench.py > profiles/r02/cfg5_shards.jsonl
"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402
from paper_1607_00291_b200 import dist as tdist  # noqa: E402
import workloads as W  # noqa: E402

PEER_GBS = 770.0


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    case = W.cfg5()
    A, B, _ = W.make_tensors(case, "cuda")
    for world in (1, 2, 4, 8):
        rg = tdist.shard_ranges(world, 0, case.lens, "abc")
        shape = tdist.shard_shape(case.lab_c, case.lens, rg)
        Cs = W.colmajor_view(torch.empty(math.prod(shape), dtype=torch.float64, device="cuda"), shape)
        As, Bs = tdist.narrow(A, case.lab_a, rg), tdist.narrow(B, case.lab_b, rg)
        info = tc.Plan.for_tensors(case.spec, As, Bs, Cs).info()
        reps = 2 if world <= 2 else 4
        ms = timed(lambda: tc.contract(case.spec, As, Bs, Cs), reps)
        m, n, k = info["m"], info["n"], info["k"]
        fl = 2.0 * m * n * k
        Ga = torch.randn(m, k, dtype=torch.float64, device="cuda")
        Gb = torch.randn(k, n, dtype=torch.float64, device="cuda")
        Gc = torch.empty(m, n, dtype=torch.float64, device="cuda")
        gms = timed(lambda: torch.mm(Ga, Gb, out=Gc), reps)
        del Ga, Gb, Gc, Cs
        torch.cuda.empty_cache()
        traffic = None if world == 1 else tdist.plan_traffic(
            world, case.lens, "abc", [(case.lab_a, 8), (case.lab_b, 8)])
        dist_ms = None if traffic is None else traffic["src_egress"] / (PEER_GBS * 1e9) * 1e3
        print(json.dumps({
            "world": world, "shard_mnk": [m, n, k], "shard_ms": round(ms, 2),
            "shard_tflops": round(fl / ms / 1e9, 2), "dgemm_tflops": round(fl / gms / 1e9, 2),
            "vs_dgemm": round(gms / ms, 3),
            "projected_job_tflops": round(world * fl / ms / 1e9, 2),
            "distribution_src_egress_gb": None if traffic is None else round(traffic["src_egress"] / 1e9, 2),
            "distribution_recv_per_rank_gb": None if traffic is None else round(max(traffic["recv"]) / 1e9, 2),
            "distribution_ms_at_770GBs": None if dist_ms is None else round(dist_ms, 1)}), flush=True)


if __name__ == "__main__":
    main()
