#!/usr/bin/env python
"""Quick A/B timing on the GPU box: per (op, bits) mean ms over R launches
(CUDA events), paper batch 2^32 bits per operand.  Not a bench line.
Usage: quick_time.py [--ops a,b] [--bits 4096,32768] [--reps 20]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_14642_b200 import bn, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="add,mul_classical,mul_ntt")
ap.add_argument("--bits", default="4096")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
dev = torch.device("cuda:0")
bn.prepare(0)
for bits in [int(x) for x in args.bits.split(",")]:
    m, n = bits // 32, (1 << 32) // bits
    a, b = inputs.make_operands(n, m, seed=1, cls="U", device=dev)
    o1 = torch.empty_like(a)
    o2 = torch.empty((n, 2 * m), dtype=a.dtype, device=dev)
    for op in args.ops.split(","):
        top = bn.ADD_BIG_MAX_BITS if op == "add_big" else bn.max_bits(op)
        if bits > top:
            continue
        f = getattr(bn, op)
        o = o2 if "wide" in op else o1
        kw = {"workspace": bn.poly_workspace(op, a)} if op.startswith("poly") else {}
        reps = args.reps if not (("classical" in op) and bits > 32768) else 3
        for _ in range(3):
            f(a, b, out=o, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f(a, b, out=o, **kw)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"op": op, "bits": bits, "ms": round(e0.elapsed_time(e1) / reps, 4)}), flush=True)
