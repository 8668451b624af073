#!/usr/bin/env python
"""Group an ncu source page (SASS) into runs of equal execution count (basic blocks)
and print the heaviest: share of executed warp instructions and of stall samples.

  ncu -i rep --page source --csv --print-source sass > x.csv; python scripts/sass_blocks.py x.csv [N]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h, rows = rows[k], rows[k + 1:]
    iA, iS, iE, iW = (h.index(x) for x in ("Address", "Source", "Instructions Executed",
                                          "Warp Stall Sampling (All Samples)"))
    blocks, cur = [], None
    for r in rows:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        w = int(r[iW]) if r[iW].isdigit() else 0
        toks = r[iS].split()
        op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")).split(".")[0]
        if cur and cur["n"] == n:
            cur["len"] += 1
            cur["ops"][op] += 1
            cur["samples"] += w
        else:
            cur = {"start": r[iA], "n": n, "len": 1, "ops": collections.Counter([op]), "samples": w}
            blocks.append(cur)
    tot = sum(b["n"] * b["len"] for b in blocks)
    ts = max(1, sum(b["samples"] for b in blocks))
    print(f"total warp instructions {tot}, stall samples {ts}")
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    for b in sorted(blocks, key=lambda b: -b["n"] * b["len"])[:top]:
        print(f"{b['start']:>8} x{b['n']:<10} len {b['len']:<4} {b['n'] * b['len'] / tot * 100:5.1f}% instr "
              f"{b['samples'] / ts * 100:5.1f}% samples  {dict(b['ops'].most_common(7))}")


if __name__ == "__main__":
    main()
