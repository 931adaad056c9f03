#!/usr/bin/env python3
"""Per-kernel pipe utilisation from ncu --set full reports -> profiles/ncu_pipes.json
(bench.py copies it into its JSON line as "ncu_pipes": the integer-pipe / tensor-pipe share of
peak for every kernel of the step, measured once per change).

  ncu_pipes.py <out.json> <report.ncu-rep | raw.csv> [...]   (.csv = ncu -i rep --page raw --csv)
"""
import csv
import io
import json
import subprocess
import sys

M = {
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "tensor_math_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_pipe_pct": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "duration_us": "gpu__time_duration.sum",
    "grid": "launch__grid_size",
    "registers": "launch__registers_per_thread",
    "smem_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_lsu_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
}


def main():
    out = {"_source": "ncu --clock-control none (pipe/dram metrics), one launch per kernel of bench.py's step: " + " ".join(sys.argv[2:]),
           "kernels": {}}
    for rep in sys.argv[2:]:
        if rep.endswith(".csv"):
            txt = open(rep).read()
        else:
            txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0].replace("Params<761, 4591, 286, 3>", "P761")
            d = {}
            for k, m in M.items():
                if m in h:
                    i = h.index(m)
                    v = float(r[i].replace(",", ""))
                    u = units[i]
                    if k.startswith("dram"):
                        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    if k == "duration_us":
                        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(u, 1)
                    d[k] = round(v, 3)
            e = out["kernels"].setdefault(name, {"launches": 0, "time_weighted": {}, "largest_launch": None})
            e["launches"] += 1
            w = d.get("duration_us", 0)
            for k in ("issue_active_pct", "alu_pipe_pct", "fma_pipe_pct", "tensor_math_pct", "tc_pipe_pct",
                      "smem_lsu_wavefronts_pct", "smem_tc_wavefronts_pct"):
                if k in d:
                    e["time_weighted"][k] = e["time_weighted"].get(k, 0) + w * d[k]
            e["_w"] = e.get("_w", 0) + w
            if e["largest_launch"] is None or w > e["largest_launch"].get("duration_us", 0):
                e["largest_launch"] = d
    for e in out["kernels"].values():
        wt = e.pop("_w", 0) or 1
        e["time_weighted"] = {k: round(v / wt, 2) for k, v in e["time_weighted"].items()}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
