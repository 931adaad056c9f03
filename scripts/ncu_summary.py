#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into text for profiles/.

  ncu_summary.py launches <launches.csv>      per-kernel launch count, device time, share
  ncu_summary.py full <report.ncu-rep>        key counters per captured launch
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("sntrup::", "").replace("Params<761, 4591, 286, 3>", "P761")
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
              "second": 1e9}.get(r[ui], 1)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print("%d launches, %.3f ms total device time (ncu: serialised, cold cache)" % (
        sum(a[0] for a in agg.values()), tot / 1e6))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%-60s %5d %10.3f ms %6.1f%%" % (k[:60], a[0], a[1] / 1e6, 100 * a[1] / tot))


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                print("%-70s %s %s" % (m, r[i], units[i] if m != "Kernel Name" else ""))
        print("---")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
