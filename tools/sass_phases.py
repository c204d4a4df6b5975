#!/usr/bin/env python
"""Split an ncu source-page export (--page source --csv --print-source sass,
optionally .gz) into phases at BAR.SYNC / BAR / WARPSYNC-free barriers and
report, per phase: stall samples, their top reasons, executed instructions,
and the opcode mix.  Usage: sass_phases.py src.csv[.gz] [min_share]"""
import collections
import csv
import gzip
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    return rows[1], rows[2:]


def main():
    path = sys.argv[1]
    min_share = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    hdr, data = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    total = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    phases, cur = [], {"start": 0, "rows": []}
    for k, r in enumerate(data):
        cur["rows"].append(r)
        src = r[ix["Source"]].strip()
        if src.startswith("BAR.SYNC") or src.startswith("BAR.RED") or src.startswith("BAR.ARV") or \
                src.startswith("UCGABAR") or src.startswith("CCTL") or " EXIT" in src or src.startswith("EXIT"):
            phases.append(cur)
            cur = {"start": k + 1, "rows": []}
    phases.append(cur)
    for p in phases:
        rows = p["rows"]
        if not rows:
            continue
        s = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows)
        if s < min_share * total:
            continue
        st = collections.Counter()
        for r in rows:
            for c in stall_cols:
                st[c] += int(r[ix[c]] or 0)
        ops = collections.Counter()
        ex = 0
        for r in rows:
            n = int(r[ix["Instructions Executed"]] or 0)
            ex += n
            opc = r[ix["Source"]].split()
            if opc:
                o = opc[0]
                if o.startswith("@"):
                    o = opc[1] if len(opc) > 1 else o
                ops[o.split(".")[0] if not o.startswith("IMAD") else o] += n
        print("phase rows %d..%d  samples %.1f%%  inst %d  last: %s" % (
            p["start"], p["start"] + len(rows) - 1, 100.0 * s / total, ex, rows[-1][ix["Source"]].strip()[:40]))
        print("   stalls:", ", ".join("%s %.0f%%" % (c[6:], 100.0 * v / max(s, 1)) for c, v in st.most_common(5)))
        print("   ops:", ", ".join("%s %.0f%%" % (o, 100.0 * v / max(ex, 1)) for o, v in ops.most_common(8)))


if __name__ == "__main__":
    main()
