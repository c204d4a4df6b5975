#!/usr/bin/env python
"""Summarise an ncu --set full report: headline metrics, pipe utilisation,
stall reasons, DRAM bytes, bank conflicts.  Usage: ncu_summary.py rep [rep...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def main():
    for rep in sys.argv[1:]:
        hdr, units, vals = raw(rep)
        for v in vals:
            d = dict(zip(hdr, v))
            u = dict(zip(hdr, units))
            print("== %s :: %s" % (rep, d.get("Kernel Name", "?")[:90]))
            for k in KEYS:
                if k in d:
                    print("  %-62s %s %s" % (k, d[k], u[k]))
            pipes = [(k, d[k]) for k in hdr if k.startswith("sm__inst_executed_pipe_") and
                     k.endswith("avg.pct_of_peak_sustained_active")]
            for k, x in sorted(pipes, key=lambda kv: -float(kv[1] or 0))[:8]:
                print("  pipe %-57s %s %%" % (k[len("sm__inst_executed_pipe_"):], x))
            st = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and
                  k.endswith("_per_issue_active.ratio")]
            tot = [(k, float(x)) for k, x in st if x not in ("", "n/a")]
            for k, x in sorted(tot, key=lambda kv: -kv[1])[:10]:
                print("  stall/issue %-50s %.2f" % (k.replace("smsp__average_warps_issue_stalled_", "")
                                                     .replace("_per_issue_active.ratio", ""), x))

if __name__ == "__main__":
    main()
