"""Summarise ncu reports / launch lists into small text files for profiles/.

usage:
  python tools/ncu_summary.py report <file.ncu-rep>       # per-kernel key metrics + stall reasons
  python tools/ncu_summary.py launches <launches.csv>     # per-kernel launch-time shares
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg", "tensor_pipe_active_pct"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_smem_active_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
]


def report(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})\n"
    h, units = rows[0], rows[1]
    out = [f"# {path}"]
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        out.append(f"\n## {name}")
        for k, label in KEYS:
            if k in h and row[h.index(k)] not in ("", "n/a"):
                out.append(f"  {label:26s} {row[h.index(k)]} {units[h.index(k)]}")
        st = [(h[i], row[i]) for i in range(len(h))
              if "smsp__average_warps_issue_stalled" in h[i] and h[i].endswith("_per_issue_active.ratio")]
        st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(v or 0)) for k, v in st), key=lambda x: -x[1])[:8]
        out.append("  stalls/issue: " + ", ".join(f"{k}={v:.2f}" for k, v in st))
    return "\n".join(out) + "\n"


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"]
    if not hi:
        return f"(no launches in {path})\n"
    h = rows[hi[0]]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi[0] + 1:]:
        if len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[h.index("Kernel Name")].split("(")[0]
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        v = v / 1000.0 if unit in ("nsecond", "ns") else v * 1000.0 if unit in ("msecond", "ms") else v
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values()) or 1.0
    out = [f"# {path} (ncu --metrics gpu__time_duration.sum; cold-cache, serialised: compare shares)",
           f"{'kernel':45s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:45s} {cnt[k]:8d} {v / cnt[k]:10.2f} {100 * v / s:6.1f}%")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    sys.stdout.write(report(path) if mode == "report" else launches(path))
