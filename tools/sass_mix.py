#!/usr/bin/env python
"""Executed-instruction mix of a kernel from an ncu report's SASS source page.
Usage: sass_mix.py report.ncu-rep  -> warp instructions per opcode (and class)."""
import collections
import csv
import io
import subprocess
import sys

FMAHEAVY = ("IMAD", "IMUL")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ie = hdr.index("Instructions Executed")
    src = hdr.index("Source")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in rows[1:]:
        op = r[src].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        n = int(r[ie] or 0)
        mix[o] += n
        stall[o] += int(r[st] or 0)
        tot += n
    print("total warp instructions %d" % tot)
    for o, n in mix.most_common(40):
        print("%-22s %12d  %5.1f%%  stall-samples %d" % (o, n, 100.0 * n / tot, stall[o]))


if __name__ == "__main__":
    main(sys.argv[1])
