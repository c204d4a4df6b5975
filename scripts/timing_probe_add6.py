#!/usr/bin/env python
"""Why the bench's per_size 6-Add is slower than quick_time's: the same op
timed (a) one event pair around 100 launches, one input; (b) bench.py's
time_op (event pair per launch, three seeds rotated); (c) (b) right after
~1 s of NTT products.  Not a bench line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_14642_b200 import bn, inputs  # noqa: E402

dev = torch.device("cuda:0")
bn.prepare(0)
st = torch.cuda.current_stream()
for bits in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32768,262144").split(",")]:
    m, n = bits // 32, (1 << 32) // bits
    ab = [inputs.make_operands(n, m, seed=s, cls="U", device=dev) for s in (1, 2, 3)]
    o = torch.empty_like(ab[0][0])
    f = lambda k: bn.add6(*ab[k % 3], out=o)  # noqa: E731
    for _ in range(3):
        f(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        f(0)
    e1.record()
    torch.cuda.synchronize()
    a = e0.elapsed_time(e1) / 100
    b = bench.stats(bench.time_op(torch, f, st, per_rep=True))["ms"]
    for _ in range(150):
        bn.mul_ntt(*ab[0], out=o)
    c = bench.stats(bench.time_op(torch, f, st, per_rep=True))["ms"]
    e0.record()
    for k in range(100):
        f(k)
    e1.record()
    torch.cuda.synchronize()
    d = e0.elapsed_time(e1) / 100  # one pair, seeds rotated
    g = bench.stats(bench.time_op(torch, lambda k: f(0), st, per_rep=True))["ms"]  # pairs, one seed
    print(json.dumps({"bits": bits, "one_pair_ms": round(a, 4), "time_op_ms": round(b, 4),
                      "after_ntt_ms": round(c, 4), "one_pair_rot_ms": round(d, 4),
                      "time_op_one_seed_ms": round(g, 4)}), flush=True)
