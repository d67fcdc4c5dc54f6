"""Summarise ncu outputs into profiles/: the per-kernel share of one epoch
(from the gpu__time_duration launch list, cold-cache and serialised) and the
key counters of each --set full capture (.ncu-rep).

    python scripts/ncu_summary.py gpurun_out/launches_c2.csv gpurun_out/prof_*.ncu-rep > profiles/x.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Instructions", "Registers Per Thread", "Achieved Occupancy",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct"]


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[r[idi]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
        names[r[idi]] = r[ki]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3, "msecond": 1e3}
    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        v, u = m["gpu__time_duration.sum"]
        t = v * scale.get(u, 1.0)
        b = sum(m[k][0] * bscale.get(m[k][1], 1) for k in ("dram__bytes_read.sum",
                                                            "dram__bytes_write.sum") if k in m)
        n = names[i].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        a = agg[n]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    print(f"### {path}: {len(per)} launches, {tot / 1e3:.2f} ms serialised\n")
    print("| kernel | launches | ms | share | DRAM GB | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{n[:70]}` | {a[0]} | {a[1] / 1e3:.2f} | {a[1] / tot:.1%} | {a[2] / 1e9:.2f} | "
              f"{a[2] / (a[1] * 1e-6) / 1e9:.0f} |")
    print()


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    kern = {}
    for row in r[1:]:
        i = row[h.index("ID")]
        kern.setdefault(i, {"name": row[h.index("Kernel Name")].split("(")[0]})
        n = row[h.index("Metric Name")]
        if n in KEYS:
            kern[i][n] = f"{row[h.index('Metric Value')]} {row[h.index('Metric Unit')]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    stalls = [c for c in rh if c.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not c.endswith("_not_issued")]
    for j, row in enumerate(rr[2:]):
        k = kern.get(row[rh.index("ID")]) if "ID" in rh else None
        if k is None:
            continue
        for c in RAW:
            if c in rh:
                k[c] = f"{row[rh.index(c)]} {rr[1][rh.index(c)]}"
        top = sorted(((float(row[rh.index(c)] or 0), c) for c in stalls), reverse=True)[:4]
        k["top stalls"] = ", ".join(f"{c.replace('smsp__pcsamp_warps_issue_stalled_', '')}"
                                    f"={v:.0f}" for v, c in top)
    print(f"### {path}\n")
    for i, k in kern.items():
        print(f"- launch {i} `{k.pop('name').replace('void ', '')}`")
        for a, b in k.items():
            print(f"  - {a}: {b}")
    print()


for p in sys.argv[1:]:
    (launch_list if p.endswith(".csv") else report)(p)
