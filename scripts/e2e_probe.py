#!/usr/bin/env python
"""bn_run_host pipeline probe: the bench step's three ops at 4096 bits over
2^20 instances through pinned host buffers, ms per call (best / median of
5).  Not a bench line."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_14642_b200 import bn, inputs  # noqa: E402

bn.prepare(0)
m, n = 128, 1 << 20
a, b = inputs.make_operands(n, m, seed=1, cls="U")
ah, bh = a.pin_memory(), b.pin_memory()
outs = [torch.empty((n, m), dtype=torch.int32, pin_memory=True) for _ in range(3)]
names = ["add", "mul_classical", "mul_ntt"]
bn.run_host(names, ah, bh, outs)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    bn.run_host(names, ah, bh, outs)
    ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"lib": os.environ.get("BN_LIB_PATH", "in-tree"), "best_ms": round(min(ts), 2),
                  "median_ms": round(statistics.median(ts), 2)}), flush=True)
