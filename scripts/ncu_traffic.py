#!/usr/bin/env python3
"""From an ncu launch list with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum, write profiles/roofline_traffic.json: per kernel kind (int8 / fp4 tensor
ring products, sampler, divsteps, encoder, ...) the average DRAM bytes and device time per launch,
and each kind's share of the device time.  bench.py reads per_launch_bytes for its roofline
"traffic" field.

  ncu_traffic.py <launches.csv> <out.json> [--skip-launches N]
"""
import collections
import csv
import json
import sys


def klass(name):
    if "tc_mul_kernel" in name or "ring_mul_kernel" in name:
        return "r3_mul" if ("Params<761, 4591, 286, 3>, 3," in name or ", 3, " in name.split(">, ")[1][:4]) else "rq_mul"
    for k in ("sample_kernel", "divstep", "joint_roots", "encode_kernel", "repair_kernel"):
        if k in name:
            return k
    return "other"


def main():
    path, out = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = r[idi]
        d = per.setdefault(key, {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        v *= {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
              "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r[mi]] = v
    agg = collections.defaultdict(lambda: {"launches": 0, "bytes": 0.0, "s": 0.0})
    for d in per.values():
        name = d["name"]
        if "tc4_mul_kernel" in name:
            c = "tc_fp4"
        elif "tc_mul_kernel" in name:
            c = "tc_int8"
        elif "ring_mul_kernel" in name:
            c = "int32"
        else:
            c = klass(name)
        a = agg[c]
        a["launches"] += 1
        a["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a["s"] += d.get("gpu__time_duration.sum", 0)
    tot = sum(a["s"] for a in agg.values())
    res = {"_source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (serialised, cold cache) on " + path,
           "per_launch_bytes": {c: a["bytes"] / a["launches"] for c, a in agg.items()},
           "per_launch_ms": {c: 1e3 * a["s"] / a["launches"] for c, a in agg.items()},
           "launches": {c: a["launches"] for c, a in agg.items()},
           "share_of_device_time": {c: a["s"] / tot for c, a in agg.items()}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
