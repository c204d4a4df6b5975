"""Host-side cost per call (tiny batch: 1 instance of 1024 bits), us."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_14642_b200 import bn, inputs
bn.prepare(0)
a, b = inputs.make_operands(1, 32, device="cuda")
o = torch.empty_like(a)
for name in ("add", "mul_classical", "mul_ntt"):
    f = getattr(bn, name)
    for _ in range(100):
        f(a, b, out=o)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        f(a, b, out=o)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print({"op": name, "host_us_per_call": (t1 - t0) / 2000 * 1e6})
