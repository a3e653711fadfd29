"""Markdown summary of one kernel from an `ncu --set full` report: time,
DRAM traffic, pipe utilisation, issue activity, L2 hit rate and the stall
breakdown of the sampled warps.   usage: python scripts/ncu_report.py rep.ncu-rep"""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main():
    rep = sys.argv[1]
    v, u = raw(rep)
    keys = [
        ("Kernel Name", "kernel"),
        ("gpu__time_duration.sum", "duration"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (realtime)"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % active"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % active"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (conversion) pipe % active"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC per SM"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ]
    print("| metric | value |\n|---|---|")
    for k, name in keys:
        if k in v:
            print(f"| {name} | {v[k]} {u.get(k, '')} |")
    stalls = {k: v[k] for k in v if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued")}
    tot = sum(float(x or 0) for x in stalls.values()) or 1.0
    print("\nSampled warp states (all warps of the CTA, incl. idle producer warps):\n")
    print("| state | share |\n|---|---|")
    for k, x in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:8]:
        print(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * float(x or 0) / tot:.1f}% |")


if __name__ == "__main__":
    main()
