#!/usr/bin/env python
"""Timing-protocol probe (not a bench line): per op and size, the mean launch
time (a) with one event pair around 100 back-to-back launches on one input,
(b) the same with the three seeds rotated, (c) bench.py's time_op (one event
pair per launch, seeds rotated).  Usage: timing_probe.py op[,op] bits[,bits]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_14642_b200 import bn, inputs  # noqa: E402

bn.prepare(0)
st = torch.cuda.current_stream()
for bits in [int(x) for x in sys.argv[2].split(",")]:
    m, n = bits // 32, (1 << 32) // bits
    ab = [inputs.make_operands(n, m, seed=s, cls="U", device=torch.device("cuda:0")) for s in (1, 2, 3)]
    o = torch.empty_like(ab[0][0])
    for op in sys.argv[1].split(","):
        fn = getattr(bn, op)
        f = lambda k, fn=fn: fn(*ab[k % 3], out=o)  # noqa: E731
        reps = 100 if "classical" not in op else 20
        res = {"op": op, "bits": bits}
        for name, rot in (("one_pair", False), ("one_pair_rot", True)):
            for k in range(3):
                f(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for k in range(reps):
                f(k if rot else 0)
            e1.record()
            torch.cuda.synchronize()
            res[name] = round(e0.elapsed_time(e1) / reps, 4)
        res["time_op"] = round(bench.stats(bench.time_op(torch, f, st, per_rep=True))["ms"], 4)
        print(json.dumps(res), flush=True)
