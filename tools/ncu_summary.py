"""Text summary of an `ncu --set full` report for profiles/: speed-of-light, pipes, DRAM traffic,
occupancy, warp-stall breakdown and the most-stalled SASS instructions.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/r01/xxx.txt
"""
import csv
import io
import subprocess
import sys

RAW_KEYS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def ncu(path, *args):
    return subprocess.run(["ncu", "-i", path, *args], capture_output=True, text=True).stdout


def main(path):
    out = []
    raw = list(csv.reader(io.StringIO(ncu(path, "--page", "raw", "--csv"))))
    if len(raw) >= 3:
        h, u = raw[0], raw[1]
        for row in raw[2:]:
            d = dict(zip(h, row))
            units = dict(zip(h, u))
            out.append(f"kernel: {d.get('Kernel Name', '?')[:120]}")
            for k in RAW_KEYS:
                if k in d:
                    out.append(f"  {k:70s} {d[k]:>16s} {units.get(k, '')}")
            stalls = []
            for k, v in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v.replace(",", "")), k[34:-23]))
                    except ValueError:
                        pass
            # the busiest units: every *.pct_of_peak_sustained_* throughput metric, top 20
            pk = []
            for k, v in d.items():
                if "pct_of_peak_sustained" in k and ("throughput" in k or "utilization" in k
                                                     or "_cycles_active" in k):
                    try:
                        pk.append((float(v.replace(",", "")), k))
                    except ValueError:
                        pass
            out.append("  busiest units (% of peak):")
            for v, k in sorted(pk, reverse=True)[:20]:
                out.append(f"    {k:86s} {v:7.2f}")
            for k, v in d.items():
                if k.startswith("l1tex__") and (k.endswith(".sum") and ("wavefronts" in k or
                                                "requests" in k or "sectors" in k)):
                    out.append(f"  {k:86s} {v:>16s}")
            tot = sum(s for s, _ in stalls) or 1.0
            out.append("  warp stalls (per issued instruction; share):")
            for s, name in sorted(stalls, reverse=True)[:10]:
                out.append(f"    {name:28s} {s:7.3f}  {100 * s / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(ncu(path, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        rows = [dict(zip(h, r)) for r in src[2:] if len(r) == len(h)]
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(float(r.get(key) or 0) for r in rows) or 1.0
        out.append("  most-sampled SASS instructions (share of all stall samples):")
        for r in sorted(rows, key=lambda r: -float(r.get(key) or 0))[:15]:
            out.append(f"    {100 * float(r.get(key) or 0) / tot:5.2f}%  {r['Source'][:80]}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
