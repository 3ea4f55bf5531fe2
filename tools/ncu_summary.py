"""Summarise ncu outputs for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/x.txt
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [kernel-regex] > profiles/y.txt
"""

import collections
import csv
import io
import re
import subprocess
import sys

TO_NS = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")) * TO_NS.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list ({path}): gpu__time_duration.sum, --clock-control none")
    print("# cold-cache serialised launches: compare SHARES, not absolute times")
    print(f"{'total_us':>12} {'share':>6} {'n':>5} {'avg_us':>10}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        name = re.sub(r"\(.*", "", k)[:90]
        print(f"{sum(v) / 1e3:12.1f} {100 * sum(v) / tot:5.1f}% {len(v):5d} {sum(v) / len(v) / 1e3:10.1f}  {name}")


WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_bytes.sum",
    "l1tex__t_bytes.sum",
]


def full(path, regex=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    print(f"# ncu --set full ({path})")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        if regex and not re.search(regex, name):
            continue
        print(f"\n## {re.sub(r'[(].*', '', name)}")
        for h, u, v in zip(hdr, units, r):
            if h in WANT or ("stall" in h and h.endswith("per_issue_active.ratio")):
                print(f"{h:72s} {v:>16s} {u}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
