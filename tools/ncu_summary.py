"""Summarise ncu output into the markdown kept under profiles/.

    python tools/ncu_summary.py launches <launches.csv> > profiles/rN_launches.md
    python tools/ncu_summary.py full <report.ncu-rep> > profiles/rN_kernels.md
"""

import collections
import re
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        # one row per vector-kernel family (instantiated per basis count)
        name = re.sub(r"^(k_\w+)<\d+>$", r"\1<nv>", name)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"ncu launch list (`gpu__time_duration.sum`, cold-cache, serialised): "
          f"{sum(cnt.values())} launches, {T:.1f} ms total\n")
    print("| kernel | launches | ms | share |\n|---|---:|---:|---:|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / T:.1f}% |")


KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Theoretical Occupancy",
        "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate"]


def full(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    per = collections.OrderedDict()
    rd = list(csv.reader(io.StringIO(det)))
    hdr = rd[0]
    for r in rd[1:]:
        d = dict(zip(hdr, r))
        name, mn = d.get("Kernel Name", ""), d.get("Metric Name", "")
        key = (d.get("ID", ""), name)
        if mn in KEYS:
            per.setdefault(key, {})[mn] = f"{d.get('Metric Value', '')} {d.get('Metric Unit', '')}"
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    traffic = {}
    for r in rr[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        try:
            t = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
            traffic[(d.get("ID", ""), d["Kernel Name"])] = f"{t:.3f} {u['dram__bytes_read.sum']}"
        except (KeyError, ValueError):
            pass
    for key, m in per.items():
        print(f"### `{key[1][:80]}` (ID {key[0]})\n")
        print("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in m:
                print(f"| {k} | {m[k]} |")
        if key in traffic:
            print(f"| dram__bytes_read+write | {traffic[key]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
