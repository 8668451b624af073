#!/usr/bin/env python
"""Summarise an ncu --set full report's warp-stall sampling and pipe utilisation for
one kernel into markdown (profiles/<tag>_stalls.md).

  python scripts/stall_summary.py <report.ncu-rep> <title> > profiles/<tag>_stalls.md
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, title = sys.argv[1], sys.argv[2]
    raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                     capture_output=True, text=True).stdout)))
    h, v = raw[0], raw[2]
    val = {k: x for k, x in zip(h, v)}
    src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                                      "sass"], capture_output=True, text=True).stdout)))
    sh, rows = src[1], src[2:]
    iS = sh.index("Warp Stall Sampling (All Samples)")
    reasons = collections.Counter()
    ops = collections.Counter()
    for r in rows:
        for j, name in enumerate(sh):
            if name.startswith("stall_") and "Not" not in name and r[j].isdigit():
                reasons[name[6:]] += int(r[j])
        if r[iS].isdigit():
            ins = r[1].split()
            o = ins[1] if ins and ins[0].startswith("@") else (ins[0] if ins else "?")
            ops[o.split(".")[0]] += int(r[iS])
    tot = sum(reasons.values()) or 1
    print(f"# {title}\n")
    print("ncu --set full, one launch; warp-state sampling over all warps (the producer warp included).\n")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
    print("| metric | value |\n|---|---:|")
    for k in keys:
        if k in val:
            print(f"| `{k}` | {val[k]} |")
    print("\n| stall reason | share |\n|---|---:|")
    for k, x in reasons.most_common(10):
        print(f"| {k} | {100 * x / tot:.1f} % |")
    print("\n| SASS opcode (samples) | share |\n|---|---:|")
    for k, x in ops.most_common(12):
        print(f"| {k} | {100 * x / tot:.1f} % |")


if __name__ == "__main__":
    main()
