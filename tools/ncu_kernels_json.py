#!/usr/bin/env python
"""Fold ncu --set full raw-page CSVs into profiles/ncu_kernels.json entries
"<op>@<bits>" (op = the bn.py call): kernel name, DRAM bytes per launch, FMA-heavy / ALU / issue-active
percentages and the launch duration, which bench.py's roofline reads.
Usage: ncu_kernels_json.py out.json op@bits:raw.csv [...]"""
import csv
import json
import os
import sys


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def row(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def f(d, k):
    """value in base units (bytes, microseconds, or as printed)"""
    try:
        v, u = d[k]
        return float(v) * SCALE.get(u, 1.0)
    except (KeyError, ValueError):
        return None


def main():
    out = sys.argv[1]
    data = json.load(open(out)) if os.path.exists(out) else {}
    for spec in sys.argv[2:]:
        key, path = spec.split(":", 1)
        d = row(path)
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        kname = d.get("Kernel Name", ("?", ""))[0]
        data[key] = {
            "kernel": kname.split("(")[0].replace("void ", ""),
            "dram_bytes": (rd + wr) if rd is not None and wr is not None else None,
            "duration_us": f(d, "gpu__time_duration.sum"),
            "fmaheavy_pct": f(d, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pct": f(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "registers": f(d, "launch__registers_per_thread"),
            "source": "ncu --set full --clock-control none, one launch, %s" % os.path.basename(path),
        }
    with open(out, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
