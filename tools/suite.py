"""Per-config performance table for every BASELINE.json config (not the driver's bench line):
contraction GFLOP/s through the C ABI next to cuBLAS DGEMM/SGEMM of equal M, N, K and the TTDT
comparator (permute to matricised copies + GEMM + permute back, fig:TTDT P:427-439), all timed
with CUDA events on the same stream after warm-up.

    python tools/suite.py [--only cfg2] [--reps 10] > profiles/r01/suite.jsonl
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402


def timeit(fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ttdt(case, A, B, C):
    """fig:TTDT: transpose A to (I,P), B to (P,J) matricised copies, GEMM, transpose-and-sum."""
    I = [x for x in case.lab_a if x in case.lab_c]
    J = [x for x in case.lab_b if x in case.lab_c]
    P = [x for x in case.lab_a if x in case.lab_b]
    m = math.prod(case.lens[x] for x in I)
    n = math.prod(case.lens[x] for x in J)
    k = math.prod(case.lens[x] for x in P)

    def run():
        At = A.permute(*[case.lab_a.index(x) for x in I + P]).reshape(m, k)
        Bt = B.permute(*[case.lab_b.index(x) for x in P + J]).reshape(k, n)
        Ct = (At @ Bt).reshape([case.lens[x] for x in I + J])
        perm = [(I + J).index(x) for x in case.lab_c]
        if case.beta != 0:
            C.mul_(case.beta).add_(Ct.permute(*perm), alpha=case.alpha)
        else:
            C.copy_(Ct.permute(*perm)).mul_(case.alpha)
    return run


def cases(only, family):
    if family == "all":
        return [c for f in ("baseline", "f1", "f2") for c in cases(only, f)]
    if family == "f2":
        out = [W.fig_bench(i) for i in range(24)]
    elif family == "f1":
        out = [W.rankk(i) for i in range(7)]
    else:
        out = [W.cfg1(), W.cfg2(False), W.cfg2(True), W.cfg3(False), W.cfg3(True)]
        out += [W.cfg4(i) for i in range(20)] + [W.cfg4(i, torch.float32) for i in range(20)]
        out.append(W.cfg5())
    return [c for c in out if not only or c.name.startswith(only)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--match", default="", help="regular expression on the case name")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-ttdt", action="store_true")
    ap.add_argument("--smtc", action="store_true",
                    help="also time the all-scatter ablation (TC_FORCE_PATH=scatter, per call)")
    ap.add_argument("--family", default="baseline", choices=["baseline", "f1", "f2", "all"])
    args = ap.parse_args()
    import re
    for case in cases(args.only, args.family):
        if args.match and not re.search(args.match, case.name):
            continue
        A, B, C = W.make_tensors(case, "cuda")
        if case.c_init == "nan":
            C.zero_()
        plan = tc.Plan.for_tensors(case.spec, A, B, C)
        info = plan.info()
        m, n, k = info["m"], info["n"], info["k"]
        fl = 2.0 * m * n * k
        reps = max(1, min(args.reps, int(2e12 / fl))) if fl > 2e12 else args.reps
        t = timeit(lambda: tc.contract(case.spec, A, B, C, case.alpha, case.beta), reps)
        Ga = torch.randn(m, k, dtype=case.dtype, device="cuda")
        Gb = torch.randn(k, n, dtype=case.dtype, device="cuda")
        Gc = torch.empty(m, n, dtype=case.dtype, device="cuda")
        tg = timeit(lambda: torch.mm(Ga, Gb, out=Gc), reps)
        del Ga, Gb, Gc
        row = {"config": case.name, "dtype": str(case.dtype).split(".")[-1], "mnk": [m, n, k],
               "swapped": info["swapped"], "a_vec_m": info["a_vec_m"], "b_vec_k": info["b_vec_k"],
               "ms": round(t, 4), "gflops": round(fl / t / 1e6, 1),
               "gemm_ms": round(tg, 4), "gemm_gflops": round(fl / tg / 1e6, 1),
               "vs_gemm": round(tg / t, 3),
               # compulsory HBM traffic (A, B read once, C written, read too when beta != 0)
               "hbm_gbs": round(A.element_size() * (A.numel() + B.numel() + C.numel() *
                                                     (2 if case.beta != 0 else 1)) / t / 1e6, 1),
               "force_path": os.environ.get("TC_FORCE_PATH", "")}
        if args.smtc:
            os.environ["TC_FORCE_PATH"] = "scatter"
            try:
                ts = timeit(lambda: tc.contract(case.spec, A, B, C, case.alpha, case.beta), reps)
            finally:
                del os.environ["TC_FORCE_PATH"]
            row.update(smtc_ms=round(ts, 4), smtc_gflops=round(fl / ts / 1e6, 1),
                       bsmtc_speedup_vs_smtc=round(ts / t, 3))
        if not args.no_ttdt:
            try:
                C2 = C.clone()
                run = ttdt(case, A, B, C2)
                torch.cuda.synchronize()
                base = torch.cuda.memory_allocated()
                torch.cuda.reset_peak_memory_stats()
                run()
                torch.cuda.synchronize()
                ws = torch.cuda.max_memory_allocated() - base
                tt = timeit(run, reps)
                # TTDT's extra device memory: the matricised copies of A and B and the GEMM
                # output before its transpose-and-sum (fig:TTDT); this path: 0
                row.update(ttdt_ms=round(tt, 4), ttdt_gflops=round(fl / tt / 1e6, 1),
                           speedup_vs_ttdt=round(tt / t, 3), ttdt_workspace_bytes=int(ws),
                           operand_bytes=int(A.element_size() * (A.numel() + B.numel() + C.numel())))
                del C2
            except torch.OutOfMemoryError:
                pass
        print(json.dumps(row), flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
