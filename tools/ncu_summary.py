#!/usr/bin/env python
"""Turn Nsight Compute reports brought back in gpurun_out/ into small tracked summaries.

    python tools/ncu_summary.py raw  gpurun_out/x.ncu-rep profiles/x_summary.csv
    python tools/ncu_summary.py list gpurun_out/launches.csv profiles/launches_summary.csv

`raw` keeps, per captured launch, the metrics the roofline argument uses (duration, DRAM
bytes, pipe utilisation, issue rate, stall reasons, registers, occupancy). `list` folds a
`--metrics gpu__time_duration.sum` launch list into per-kernel totals and shares.
"""

from __future__ import annotations

import csv
import re
import subprocess
import sys
from collections import OrderedDict

KEEP = [
    "gpu__time_duration.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"snt::", "", name)
    return re.sub(r"\(.*", "", name)[:90]


def raw(rep: str, out: str) -> None:
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(text.splitlines()) if r]
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [c for c in KEEP if c in hdr]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + cols)
        w.writerow(["unit"] + [units[hdr.index(c)] for c in cols])
        for r in data:
            w.writerow([short(r[hdr.index("Kernel Name")])] + [r[hdr.index(c)] for c in cols])
    print(f"wrote {out}: {len(data)} launch(es), {len(cols)} metrics")


def launch_list(src: str, out: str) -> None:
    rows = [r for r in csv.reader(open(src)) if len(r) > 8]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "nsecond": 1e-3}.get(r[ui], 1.0)
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(a[1] for a in agg.values())
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "avg_us", "share_of_listed_time"])
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, n, f"{t:.1f}", f"{t / n:.2f}", f"{t / total:.4f}"])
    print(f"wrote {out}: {len(agg)} kernels, {total:.0f} us listed")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (raw if mode == "raw" else launch_list)(src, dst)
