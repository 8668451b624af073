#!/usr/bin/env python
"""Summarise gpurun_out/ ncu artefacts into tracked files under profiles/.

  python scripts/summarize_profiles.py <round-tag> [suffix]

suffix (e.g. _fp8) selects the files profile_box.sh wrote with TAG=<suffix>.

Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch list of
`bench.py --profile`) and gpurun_out/prof_{realign,match}.ncu-rep (ncu --set full),
writes profiles/<tag>_launches.md, profiles/<tag>_ncu_<kernel>.txt and
profiles/realign_ncu.json (per-launch DRAM traffic that bench.py reports).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def realign_src_hash():
    """sha256 of the sources that define the realign kernel (bench.py computes the same
    hash and reports the committed DRAM traffic only for the build it was captured on)."""
    import hashlib
    h = hashlib.sha256()
    for f in ("realign.cu", "kvcomm_internal.h", "ptx.cuh", "Makefile"):
        h.update(open(os.path.join(ROOT, "paper_2510_12872_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(unit, v)


def launches(tag, sfx=""):
    path = os.path.join(OUT, f"launches{sfx}.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += to_us(r[vi], r[ui])
    tot = sum(v[1] for v in agg.values())
    steps = json.loads(open(os.path.join(OUT, f"launches{sfx}.log")).read().strip().splitlines()[-1]).get("profile_steps", 1)
    lines = [f"# {tag}: kernel launch list of `bench.py --profile` ({steps} steps)", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off "
             "(serialised, cold-cache per launch: compare SHARES, not absolutes).", "",
             "| kernel | launches | total us | us / step | share |", "|---|---:|---:|---:|---:|"]
    for n, (c, t) in agg.items():
        lines.append(f"| `{n}` | {c} | {t:.1f} | {t / steps:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| **all** | {sum(v[0] for v in agg.values())} | {tot:.1f} | {tot / steps:.1f} | 100% |")
    open(os.path.join(PROF, f"{tag}{sfx}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for i, n in enumerate(hdr):
            if n in RAW_KEYS or n in ("Kernel Name", "ID"):
                d[n] = (r[i], units[i])
        out.append(d)
    return out


def details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
            "Warp State Statistics", "Scheduler Statistics")
    lines = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Section Name") in keep:
            lines.append(f"{d['ID']:>3} {d['Section Name'][:28]:28s} {d['Metric Name'][:48]:48s} "
                         f"{d['Metric Value']:>16s} {d['Metric Unit']}")
    return lines


def kernel_summary(tag, name, sfx=""):
    rep = os.path.join(OUT, f"prof_{name}{sfx}.ncu-rep")
    if not os.path.exists(rep):
        return None
    rs = raw(rep)
    lines = [f"# {tag}: ncu --set full of {name} ({len(rs)} launch(es))", ""]
    for d in rs:
        lines.append(f"## launch ID {d.get('ID', ('?',))[0]}: {d.get('Kernel Name', ('?',))[0]}")
        for k in RAW_KEYS:
            if k in d:
                lines.append(f"{k:60s} {d[k][0]:>20s} {d[k][1]}")
        lines.append("")
    lines += ["## details", ""] + details(rep)
    open(os.path.join(PROF, f"{tag}{sfx}_ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
    return rs


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    sfx = sys.argv[2] if len(sys.argv) > 2 else ""
    os.makedirs(PROF, exist_ok=True)
    launches(tag, sfx)
    rs = kernel_summary(tag, "realign", sfx)
    kernel_summary(tag, "match", sfx)
    if rs:
        d = rs[0]

        def val(k, scale):
            v, u = d[k]
            v = float(v.replace(",", ""))
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0) * scale

        rd, wr = val("dram__bytes_read.sum", 1), val("dram__bytes_write.sum", 1)
        t_ms = to_us(*d["gpu__time_duration.sum"]) / 1e3
        js = {"source": f"profiles/{tag}{sfx}_ncu_realign.txt (ncu --set full, 1 launch, bench.py --profile)",
              "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
              "duration_ms_under_ncu": t_ms, "dram_gbs_under_ncu": (rd + wr) / (t_ms / 1e3) / 1e9,
              "realign_src_sha": realign_src_hash()}
        json.dump(js, open(os.path.join(PROF, f"realign_ncu{sfx}.json"), "w"), indent=1)
        print(json.dumps(js, indent=1))


if __name__ == "__main__":
    main()
