#!/usr/bin/env python
"""Side-by-side of our B200 numbers (a bench line's per_size, or the round-1
sweep profiles/r01_sweep.jsonl) with the paper's
A100 numbers (BASELINE.md Tables 1-2) —
context only: other hardware, and the paper's FFT digit scheme is inexact
(reading R10).  Prints a markdown table."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# bits -> (Our-CUDA 1-Add GB/s, 6-Add GB/s, CUDA-Quad 1-Mul, CUDA-FFT 1-Mul, Quad Poly, FFT Poly) [Gu32ops/s]
PAPER = {
    2048: (1366, 855, 70661, 13554, 60819, 10884),
    4096: (1359, 856, 49328, 15264, 42673, 11189),
    8192: (1350, 816, 31658, 15791, 27876, 15173),
    16384: (1334, 836, 21608, 14297, 19455, 13899),
    32768: (1363, 856, 13460, 12779, 12247, 12621),
    65536: (1358, 853, 7843, 11466, 7148, 11679),
    131072: (1331, 803, 4471, 11789, 4027, 12130),
    262144: (1320, 570, None, 11590, None, 11351),
}


def _from_bench_line(line):
    """rows of the sweep format from a bench line's per_size block; Poly
    Gu32ops/s = 4 multiplications x the paper's 1-Mul u32-op count
    (300 m log2 m) per instance"""
    import math
    rows = []
    for bits, row in line["per_size"].items():
        if not bits.isdigit():
            continue
        b, m = int(bits), int(bits) // 32
        for op, r in row.items():
            if not isinstance(r, dict):
                continue
            r = dict(r, op=op, bits=b)
            if op.startswith("poly") and "poly/s" in r:
                r["Gu32ops/s"] = r["poly/s"] * 4 * 300 * m * math.log2(m) / 1e9
            rows.append(r)
    return rows


def main(path=os.path.join(ROOT, "profiles", "r01_sweep.jsonl")):
    """path: a --sweep JSONL (round 1) or a bench JSON line with per_size"""
    lines = [json.loads(l) for l in open(path) if l.strip()]
    rows = _from_bench_line(lines[-1]) if "per_size" in lines[-1] else lines
    by = {}
    for r in rows:
        by.setdefault(r["op"], {})[r["bits"]] = r
    cols = [("add", "GB/s", 0), ("add6", "GB/s", 1), ("mul_classical", "Gu32ops/s", 2),
            ("mul_ntt", "Gu32ops/s", 3), ("poly_classical", "Gu32ops/s", 4), ("poly_ntt", "Gu32ops/s", 5)]
    print("| bits | " + " | ".join("%s B200 / A100" % c for c, _, _ in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for bits in sorted(PAPER):
        cells = []
        for op, key, i in cols:
            ours = by.get(op, {}).get(bits, {}).get(key)
            paper = PAPER[bits][i]
            if ours is None or paper is None:
                cells.append("%s / %s" % ("%.0f" % ours if ours else "-", paper or "n/a"))
            else:
                cells.append("%.0f / %d (%.1fx)" % (ours, paper, ours / paper))
        print("| %d | %s |" % (bits, " | ".join(cells)))


if __name__ == "__main__":
    main(*sys.argv[1:])
