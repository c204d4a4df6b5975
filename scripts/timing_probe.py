#!/usr/bin/env python
"""Does the per_size timing (one event pair per launch, seeds rotated) differ
from back-to-back launches on one buffer?  Prints ms per launch for the four
combinations, for a few (op, bits)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_14642_b200 import bn, inputs  # noqa: E402

dev = torch.device("cuda:0")
bn.prepare(0)
for op, bits in (("add", 4096), ("add6", 16384), ("add6", 32768), ("add6", 262144), ("mul_ntt", 4096)):
    m, n = bits // 32, (1 << 32) // bits
    ab = [inputs.make_operands(n, m, seed=s, cls="U", device=dev) for s in (1, 2, 3)]
    o = torch.empty_like(ab[0][0])
    f = getattr(bn, op)
    reps = 60
    for rot in (False, True):
        for per_launch in (False, True):
            for k in range(3):
                f(*ab[k % 3], out=o)
            torch.cuda.synchronize()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
            evs[0].record()
            for k in range(reps):
                x, y = ab[k % 3] if rot else ab[0]
                f(x, y, out=o)
                if per_launch:
                    evs[k + 1].record()
            if not per_launch:
                evs[reps].record()
            torch.cuda.synchronize()
            ms = evs[0].elapsed_time(evs[reps]) / reps
            print(json.dumps({"op": op, "bits": bits, "rotate_seeds": rot, "event_per_launch": per_launch,
                              "ms": round(ms, 4)}), flush=True)
    del ab, o
    torch.cuda.empty_cache()
