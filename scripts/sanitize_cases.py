"""Small invocations of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): every op at small and large sizes up to
its maximum (fused and wide products to 256K bits), ragged batches, a grid
cap so the persistent paths run, and (--big) the cluster sizes 512K / 1M.  Results are checked against the oracle (any mismatch exits 1).
SAN_OPS=key[,key] restricts the run to those result keys (add, mul, add6,
poly, wide)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2405_14642_b200 import bn, inputs  # noqa: E402

dev = torch.device("cuda:0")
bn.prepare(0)
bad = 0
cases = [(1024, 37), (2048, 41), (4096, 19), (65536, 3), (131072, 2), (262144, 1)]
if "--big" in sys.argv:
    cases += [(1 << 19, 2), (1 << 20, 1), (1 << 22, 2)]
for cap in (0, 2):
    bn.debug_set_grid_cap(cap)
    for bits, n in cases:
        m = bits // 32
        a, b = inputs.make_operands(n, m, seed=bits + cap, cls="MIX")
        an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
        da, db = a.to(dev), b.to(dev)
        want = {"add": O.add(an, bnp)}
        ops = []
        if bits <= bn.max_bits("add"):
            ops += [("add", bn.add)]
        if bits <= bn.max_bits("mul_ntt"):
            want["mul"] = O.mul(an, bnp, nthreads=8)
            ops += [("mul", bn.mul_ntt)]
        if bits <= bn.max_bits("mul_classical"):
            ops += [("mul", bn.mul_classical)]
        if bits <= 262144:
            want["add6"] = O.add6(an, bnp)
            want["poly"] = O.poly(an, bnp, nthreads=8)
            want["wide"] = O.mul_full_rows(an, bnp)
            ops += [("add6", bn.add6), ("poly", bn.poly_classical), ("poly", bn.poly_ntt),
                    ("wide", bn.mul_wide_classical), ("wide", bn.mul_wide_ntt)]
        if bits >= (1 << 18):
            ops += [("add", bn.add_big)]
        only = os.environ.get("SAN_OPS")  # e.g. SAN_OPS=add6: one op key only
        for key, f in ops:
            if only and key not in only.split(","):
                continue
            got = inputs.to_numpy_u32(f(da, db))
            torch.cuda.synchronize()
            if not np.array_equal(got, want[key]):
                print("MISMATCH", f.__name__, bits, cap)
                bad += 1
bn.debug_set_grid_cap(0)
print("sanitize cases done, mismatches:", bad)
sys.exit(1 if bad else 0)
