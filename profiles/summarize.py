#!/usr/bin/env python
"""Summarise ncu output brought back by gpurun into committed text files.

    python profiles/summarize.py launches <launches.csv> > profiles/rNN/launches_summary.txt
    python profiles/summarize.py details <report.ncu-rep> > profiles/rNN/<kernel>_details.txt
    python profiles/summarize.py lines <report.ncu-rep> <kernel-regex> > profiles/rNN/<kernel>_lines.txt

``launches``: per-kernel launch counts, summed device time and share of the
captured region (ncu --metrics gpu__time_duration.sum; cold-cache and
serialised, so compare shares, not absolutes).
``details``: SpeedOfLight / occupancy / memory / warp-state figures and the
DRAM bytes per launch (the roofline ``traffic`` field) for every profiled
launch in a ``--set full`` report.
``lines``: warp-stall samples aggregated per CUDA source line (needs
-lineinfo), the hottest first.
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Occupancy", "Launch Statistics", "Compute Workload Analysis",
            "Memory Workload Analysis", "Warp State Statistics")
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Block Size", "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")


def ncu_csv(*args) -> list[list[str]]:
    out = subprocess.run(["ncu", *args], check=True, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_us(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += to_us(r[vi], r[ui])
    tot = sum(t for _, t in agg.values())
    print(f"# {path}: {sum(c for c, _ in agg.values())} launches, {tot / 1e3:.2f} ms total device time")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {c:8d} {t / 1e3:10.3f} {100 * t / tot:6.1f}%")


def details(path: str) -> None:
    rows = ncu_csv("-i", path, "--page", "details", "--csv")
    h = rows[0]
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Section Name") in SECTIONS and d.get("Metric Name") in KEEP:
            per.setdefault((d["ID"], d["Kernel Name"].split("(")[0]), []).append(
                f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}".rstrip())
    raw = ncu_csv("-i", path, "--page", "raw", "--csv")
    rh = raw[0]
    rawv = {}
    for r in raw[2:]:
        d = dict(zip(rh, r))
        rawv[d["ID"]] = {k: d.get(k) for k in RAW if k in d}
    for (i, name), lines in per.items():
        print(f"== launch {i}: {name}")
        for ln in lines:
            print("  " + ln)
        uu = dict(zip(rh, raw[1])) if len(raw) > 1 else {}
        for k, v in rawv.get(i, {}).items():
            print(f"  {k}: {v} {uu.get(k, '')}".rstrip())
        units = raw[1] if len(raw) > 1 else []
        if units:  # each metric in its own unit (ncu scales them independently)
            u = dict(zip(rh, units))
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            b = sum(float((rawv.get(i, {}).get(k) or "0").replace(",", "")) * scale.get(u.get(k, "byte"), 1.0)
                    for k in RAW[:2])
            print(f"  traffic (dram read + write): {b / 1e9:.4g} Gbyte")


def lines(path: str, kernel: str) -> None:
    rows = ncu_csv("-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}", "--launch-count", "1",
                   "--print-source", "cuda,sass")
    cur, agg, tot = None, collections.Counter(), 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 6:
            continue
        try:
            ln, s = int(r[0]), int(r[4])
        except ValueError:
            continue
        agg[(cur, ln, r[1].strip()[:80])] += s
        tot += s
    print(f"# {path} kernel {kernel}: {tot} warp-stall samples (all), by CUDA source line")
    by_file = collections.Counter()
    for (f, _, _), s in agg.items():
        by_file[f] += s
    for f, s in by_file.most_common():
        print(f"#   {f}: {100 * s / max(tot, 1):.1f}%")
    for (f, ln, src), s in agg.most_common(40):
        print(f"{100 * s / max(tot, 1):5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "details":
        details(sys.argv[2])
    elif cmd == "lines":
        lines(sys.argv[2], sys.argv[3])
    else:
        raise SystemExit(__doc__)
