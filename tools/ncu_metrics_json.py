#!/usr/bin/env python
"""Fold `ncu --metrics ... --csv` logs (one row per metric) into
profiles/ncu_kernels.json entries "<op>@<bits>" (same fields as
tools/ncu_kernels_json.py).  Usage: ncu_metrics_json.py out.json m_<op>_<bits>.csv ..."""
import csv
import io
import json
import os
import re
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
FIELDS = {"gpu__time_duration.sum": "duration_us",
          "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active": "fmaheavy_pct",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
          "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
          "launch__registers_per_thread": "registers"}


def main():
    out = sys.argv[1]
    data = json.load(open(out)) if os.path.exists(out) else {}
    for path in sys.argv[2:]:
        m = re.match(r"m_(.+)_(\d+)\.csv$", os.path.basename(path))
        if not m:
            continue
        key = "%s@%s" % (m.group(1), m.group(2))
        txt = open(path).read()
        if '"ID"' not in txt:
            continue
        rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
        if not rows:
            continue
        e = {"kernel": rows[0]["Kernel Name"].split("(")[0].replace("void ", ""),
             "source": "ncu --metrics (pipes, issue, DRAM) --clock-control none, one launch, %s" % os.path.basename(path)}
        rd = wr = None
        for r in rows:
            v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
            if r["Metric Name"] in FIELDS:
                e[FIELDS[r["Metric Name"]]] = v
            elif r["Metric Name"] == "dram__bytes_read.sum":
                rd = v
            elif r["Metric Name"] == "dram__bytes_write.sum":
                wr = v
        e["dram_bytes"] = rd + wr if rd is not None and wr is not None else None
        if key in data and "set full" in data[key].get("source", ""):
            continue  # keep the full capture
        data[key] = e
    with open(out, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
