"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle — -m gpu.

Bit-exact comparisons (integer work, zero tolerance) on seeded synthetic
inputs (paper_2405_14642_b200/inputs.py), at every supported size
2^10..2^18 bits, every input class, with batch sizes that span several CTAs
plus a ragged tail; plus the full-size bench configuration (sampled
instances vs the oracle, and whole-batch properties: classical == NTT,
closed forms for ONES / RIPPLE), u64 limbs, in-place calls, streams, the
host-buffer pipeline, and the NTT forward stage against the DFT definition.
"""
import numpy as np
import pytest
import torch

from oracle import ntt_ref as R
from oracle import oracle as O
from paper_2405_14642_b200 import bn, inputs

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
SIZES = [1 << k for k in range(10, 19)]
# several CTAs + a ragged tail for every kernel's instances-per-CTA
N_INST = {1024: 1029, 2048: 517, 4096: 261, 8192: 131, 16384: 67, 32768: 35, 65536: 13,
          131072: 5, 262144: 3}
CLASSES = ["U", "ONES", "RIPPLE", "RUNS", "SPARSE", "MIX"]
OPS = {"add": bn.add, "mul_classical": bn.mul_classical, "mul_ntt": bn.mul_ntt}


def _first_bad(got, want):
    rows = np.argwhere((got != want).any(axis=1))
    if rows.size == 0:
        return None
    i = int(rows[0][0])
    cols = np.argwhere(got[i] != want[i]).ravel()
    return "instance %d, first bad limb %d of %d (%d bad rows)" % (i, int(cols[0]), got.shape[1], rows.size)


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import __graft_entry__ as ge
    ge.build()
    torch.cuda.set_device(DEV)
    bn.prepare(0)


@pytest.mark.parametrize("cls", CLASSES)
@pytest.mark.parametrize("bits", SIZES)
def test_parity_all_ops(bits, cls):
    m = bits // 32
    n = N_INST[bits]
    a, b = inputs.make_operands(n, m, seed=bits + len(cls), cls=cls)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    want = {"add": O.add(an, bnp, nthreads=8)}
    want["mul_classical"] = want["mul_ntt"] = O.mul(an, bnp, nthreads=8)
    da, db = a.to(DEV), b.to(DEV)
    for name, f in OPS.items():
        got = inputs.to_numpy_u32(f(da, db))
        bad = _first_bad(got, want[name])
        assert bad is None, "%s %d bits %s: %s" % (name, bits, cls, bad)


@pytest.mark.parametrize("bits", [1024, 4096, 262144])
def test_single_instance_and_seeds(bits):
    m = bits // 32
    for seed in range(16 if bits <= 4096 else 2):
        a, b = inputs.make_operands(1, m, seed=seed, cls="U")
        an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
        da, db = a.to(DEV), b.to(DEV)
        assert np.array_equal(inputs.to_numpy_u32(bn.add(da, db)), O.add(an, bnp))
        w = O.mul(an, bnp)
        assert np.array_equal(inputs.to_numpy_u32(bn.mul_classical(da, db)), w)
        assert np.array_equal(inputs.to_numpy_u32(bn.mul_ntt(da, db)), w)


@pytest.mark.parametrize("bits", [1024, 2048, 65536])
def test_u64_limbs_and_in_place(bits):
    m = bits // 32
    a, b = inputs.make_operands(9, m, seed=3, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    a64, b64 = da.view(torch.int64), db.view(torch.int64)
    for name, f in OPS.items():
        want = O.add(an, bnp) if name == "add" else O.mul(an, bnp)
        got = f(a64, b64).view(torch.int32)
        assert np.array_equal(inputs.to_numpy_u32(got), want), name
        x = da.clone()
        f(x, db, out=x)  # out == a
        assert np.array_equal(inputs.to_numpy_u32(x), want), name + " in-place a"
        y = db.clone()
        f(da, y, out=y)  # out == b
        assert np.array_equal(inputs.to_numpy_u32(y), want), name + " in-place b"
        z = da.clone()
        f(z, z, out=z)  # out == a == b
        want_sq = O.add(an, an) if name == "add" else O.mul(an, an)
        assert np.array_equal(inputs.to_numpy_u32(z), want_sq), name + " in-place a == b"


def test_empty_batch_and_streams():
    z = torch.zeros((0, 32), dtype=torch.int32, device=DEV)
    assert bn.add(z, z).shape == (0, 32)
    m = 256
    a, b = inputs.make_operands(50, m, seed=5)
    da, db = a.to(DEV), b.to(DEV)
    want = O.mul(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        r1 = bn.mul_ntt(da, db)
    with torch.cuda.stream(s2):
        r2 = bn.mul_classical(da, db)
    torch.cuda.synchronize()
    assert np.array_equal(inputs.to_numpy_u32(r1), want)
    assert np.array_equal(inputs.to_numpy_u32(r2), want)


# --------------------------------------------------- full-size configurations

def _sample_check(da, db, outs, idx):
    an = inputs.to_numpy_u32(da[idx])
    bnp = inputs.to_numpy_u32(db[idx])
    wa, wm = O.add(an, bnp, nthreads=8), O.mul(an, bnp, nthreads=8)
    for name, t in outs.items():
        got = inputs.to_numpy_u32(t[idx])
        assert np.array_equal(got, wa if name == "add" else wm), name


def test_full_size_bench_config_4096():
    """BASELINE configs[1]: 4096-bit batch of 2^20 instances (the bench workload,
    same launch configuration): 512 sampled instances vs the oracle, and
    classical == NTT over the whole batch."""
    m, n = 128, 1 << 20
    a, b = inputs.make_operands(n, m, seed=1, cls="U", device=DEV)
    outs = {k: f(a, b) for k, f in OPS.items()}
    torch.cuda.synchronize()
    assert torch.equal(outs["mul_classical"], outs["mul_ntt"])
    g = torch.Generator().manual_seed(0)
    idx = torch.cat([torch.tensor([0, n - 1]), torch.randint(0, n, (510,), generator=g)]).to(DEV)
    _sample_check(a, b, outs, idx)


@pytest.mark.parametrize("bits,n", [(32768, 1 << 17), (65536, 1 << 16), (131072, 1 << 15), (262144, 1 << 14)])
def test_full_size_closed_forms(bits, n):
    """configs[2] / configs[3] / configs[4]: full paper batch (2^32 bits), worst-case all-ones
    carry chains: (2^B-1)+(2^B-1) = [FFFFFFFE, FF..], (2^B-1)^2 = 1 mod 2^B,
    (2^B-1)+1 = 0, (2^B-1)*1 = 2^B-1 — checked on every instance."""
    m = bits // 32
    ones, _ = inputs.make_operands(n, m, seed=1, cls="ONES", device=DEV)
    s = bn.add(ones, ones)
    want_s = torch.full((m,), -1, dtype=torch.int32, device=DEV)
    want_s[0] = -2
    assert torch.equal(s, want_s.expand(n, m))
    one = torch.zeros((m,), dtype=torch.int32, device=DEV)
    one[0] = 1
    for f in (bn.mul_classical, bn.mul_ntt):
        if f is bn.mul_classical and bits == 262144:
            continue  # covered by the sampled test below (quadratic: slow at full batch)
        assert torch.equal(f(ones, ones), one.expand(n, m))
    _, rip = inputs.make_operands(n, m, seed=1, cls="RIPPLE", device=DEV)
    assert not bn.add(ones, rip).any()
    assert torch.equal(bn.mul_ntt(ones, rip), ones)
    # random operands: NTT vs oracle on sampled instances
    a, b = inputs.make_operands(n, m, seed=2, cls="U", device=DEV)
    outs = {"add": bn.add(a, b), "mul_ntt": bn.mul_ntt(a, b)}
    idx = torch.tensor([0, 1, n // 2, n - 1], device=DEV)
    _sample_check(a, b, outs, idx)


@pytest.mark.parametrize("cap", [1, 3, 7])
@pytest.mark.parametrize("bits", [1024, 4096, 65536])
def test_grid_stride_paths(bits, cap):
    """Results must not depend on the launch configuration (R20): cap the grid
    so every CTA runs many groups (persistent / double-buffered paths)."""
    m = bits // 32
    n = 301 if bits <= 4096 else 9
    a, b = inputs.make_operands(n, m, seed=cap, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    wa, wm = O.add(an, bnp, nthreads=8), O.mul(an, bnp, nthreads=8)
    da, db = a.to(DEV), b.to(DEV)
    bn.debug_set_grid_cap(cap)
    try:
        got = {k: inputs.to_numpy_u32(f(da, db)) for k, f in OPS.items()}
    finally:
        bn.debug_set_grid_cap(0)
    for k, g in got.items():
        bad = _first_bad(g, wa if k == "add" else wm)
        assert bad is None, "%s cap=%d: %s" % (k, cap, bad)


def test_classical_equals_ntt_every_size():
    """Whole paper-sized batches (2^32 bits per operand) at every
    size: the two multiplication kernels agree on every instance (this is the
    configuration in which a cross-warp race once showed up, in ~0.5% of the
    instances of a 2^20 batch, while small batches passed)."""
    for bits in SIZES:
        m = bits // 32
        n = (1 << 32) // bits
        a, b = inputs.make_operands(n, m, seed=9, cls="MIX", device=DEV)
        assert torch.equal(bn.mul_classical(a, b), bn.mul_ntt(a, b)), bits


# ------------------------------------------------------------------ NTT stage

def _bitrev(i, lg):
    r = 0
    for _ in range(lg):
        r = (r << 1) | (i & 1)
        i >>= 1
    return r


@pytest.mark.parametrize("lg", [6, 7, 8, 10, 12])
@pytest.mark.parametrize("prime", [0, 1, 2])
def test_ntt_forward_stage(lg, prime):
    """DIF forward transform (debug entry point) == the DFT definition
    (O(N^2) direct for N <= 128, Fig. 9 radix-2 reference above), output in
    bit-reversed order; constants: the library's prime and omega."""
    N = 1 << lg
    p = bn.ntt_primes()[prime]
    rng = np.random.default_rng(lg * 3 + prime)
    rows = 3
    x = rng.integers(0, p, size=(rows, N), dtype=np.int64)
    x[0] = 0
    x[0, 0] = 1  # delta -> all ones
    xt = inputs.from_numpy_u32(x.astype(np.uint32), DEV)
    out, w = bn.debug_ntt_forward(xt, prime)
    got = inputs.to_numpy_u32(out).astype(np.int64)
    assert pow(w, N, p) == 1 and pow(w, N // 2, p) == p - 1
    for r in range(rows):
        xs = [int(v) for v in x[r]]
        if N <= 128:
            want = R.dft_direct(xs, w, p)
        else:
            want = R.fft_fig9(xs, R.omegas_table(p, w, N), p)
        assert [int(got[r][_bitrev(k, lg)]) for k in range(N)] == want


# ------------------------------------------------------------ host pipeline

@pytest.mark.parametrize("bits", [1024, 32768])
def test_run_host_pipeline(bits):
    m = bits // 32
    # 64 MiB per operand + a ragged tail: five 16 MiB chunks, so all three
    # pipeline streams are reused and the last chunk is partial
    n = (1 << 29) // bits + 7
    a, b = inputs.make_operands(n, m, seed=4, cls="MIX")
    a, b = a.pin_memory(), b.pin_memory()
    outs = bn.run_host(["add", "mul_classical", "mul_ntt"], a, b)
    da, db = a.to(DEV), b.to(DEV)
    assert torch.equal(outs[0], bn.add(da, db).cpu())
    wm = bn.mul_ntt(da, db).cpu()
    assert torch.equal(outs[1], wm) and torch.equal(outs[2], wm)
    idx = [0, n // 3, n - 1]
    an, bnp = inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx])
    assert np.array_equal(inputs.to_numpy_u32(outs[1][idx]), O.mul(an, bnp))


# ------------------------------------- fused workloads: 6-Add, Poly (§8(f) #1)

FUSED = {"add6": (bn.add6, O.add6), "poly_classical": (bn.poly_classical, O.poly),
         "poly_ntt": (bn.poly_ntt, O.poly)}


@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "RUNS", "MIX"])
@pytest.mark.parametrize("bits", SIZES)
def test_parity_fused(bits, cls):
    """6-Add and Poly (classical and NTT) vs the oracle's compositions,
    bit-exact, several CTAs + a ragged tail at every size."""
    m = bits // 32
    n = N_INST[bits]
    a, b = inputs.make_operands(n, m, seed=3 * bits + len(cls), cls=cls)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    want6 = O.add6(an, bnp, nthreads=8)
    wantp = O.poly(an, bnp, nthreads=8)
    for name, (f, _) in FUSED.items():
        got = inputs.to_numpy_u32(f(da, db))
        bad = _first_bad(got, want6 if name == "add6" else wantp)
        assert bad is None, "%s %d bits %s: %s" % (name, bits, cls, bad)


@pytest.mark.parametrize("cap", [1, 5])
@pytest.mark.parametrize("bits", [1024, 8192, 131072])
def test_fused_grid_cap_and_workspace_reuse(bits, cap):
    """Persistent CTAs that each run many groups reuse their workspace slice
    group after group; results must not change (R20)."""
    m = bits // 32
    n = 203 if bits <= 8192 else 7
    a, b = inputs.make_operands(n, m, seed=cap + 40, cls="MIX")
    wantp = O.poly(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b), nthreads=8)
    want6 = O.add6(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b))
    da, db = a.to(DEV), b.to(DEV)
    bn.debug_set_grid_cap(cap)
    try:
        got = {k: inputs.to_numpy_u32(f(da, db)) for k, (f, _) in FUSED.items()}
    finally:
        bn.debug_set_grid_cap(0)
    for k, g in got.items():
        bad = _first_bad(g, want6 if k == "add6" else wantp)
        assert bad is None, "%s cap=%d: %s" % (k, cap, bad)


@pytest.mark.parametrize("m", [32, 64])
def test_fused_u64_in_place_and_workspace_errors(m):
    a, b = inputs.make_operands(33, m, seed=12, cls="U")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    wantp = O.poly(an, bnp)
    for f in (bn.poly_classical, bn.poly_ntt):
        got = f(da.view(torch.int64), db.view(torch.int64)).view(torch.int32)
        assert np.array_equal(inputs.to_numpy_u32(got), wantp)
        x = da.clone()
        f(x, db, out=x)
        assert np.array_equal(inputs.to_numpy_u32(x), wantp)
    x = db.clone()
    bn.add6(da, x, out=x)
    assert np.array_equal(inputs.to_numpy_u32(x), O.add6(an, bnp))
    for op, f in (("poly_classical", bn.poly_classical), ("poly_ntt", bn.poly_ntt)):
        need = bn.poly_workspace_bytes(op, 33, m)
        assert 0 < need <= 3 * 33 * m * 4 * 2
        ws = torch.empty(need - 16, dtype=torch.uint8, device=DEV)
        with pytest.raises(bn.BnError):
            f(da, db, workspace=ws)
        ws = torch.empty(need, dtype=torch.uint8, device=DEV)
        assert np.array_equal(inputs.to_numpy_u32(f(da, db, workspace=ws)), wantp)


def test_fused_full_size_4096():
    """The fused workloads at the bench size (4096 bits, 2^20 instances):
    poly_classical == poly_ntt over the whole batch, 256 sampled instances
    vs the oracle, and 6-Add == 4a + 3b through the single-op kernels."""
    m, n = 128, 1 << 20
    a, b = inputs.make_operands(n, m, seed=5, cls="U", device=DEV)
    pc, pn = bn.poly_classical(a, b), bn.poly_ntt(a, b)
    assert torch.equal(pc, pn)
    s6 = bn.add6(a, b)
    a2 = bn.add(a, a)
    a4 = bn.add(a2, a2)
    b3 = bn.add(bn.add(b, b), b)
    assert torch.equal(s6, bn.add(a4, b3))
    g = torch.Generator().manual_seed(1)
    idx = torch.cat([torch.tensor([0, n - 1]), torch.randint(0, n, (254,), generator=g)]).to(DEV)
    an, bnp = inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx])
    assert np.array_equal(inputs.to_numpy_u32(pn[idx]), O.poly(an, bnp, nthreads=8))
    assert np.array_equal(inputs.to_numpy_u32(s6[idx]), O.add6(an, bnp))


@pytest.mark.parametrize("bits", [32768, 262144])
def test_fused_closed_forms_full_batch(bits):
    """Worst-case all-ones at the paper batch: Poly(-1, -1) = 1, 6-Add = -7."""
    m = bits // 32
    n = (1 << 32) // bits
    ones, _ = inputs.make_operands(n, m, seed=1, cls="ONES", device=DEV)
    one = torch.zeros((m,), dtype=torch.int32, device=DEV)
    one[0] = 1
    assert torch.equal(bn.poly_ntt(ones, ones), one.expand(n, m))
    minus7 = torch.full((m,), -1, dtype=torch.int32, device=DEV)
    minus7[0] = -7
    assert torch.equal(bn.add6(ones, ones), minus7.expand(n, m))


@pytest.mark.parametrize("bits", [1024, 32768])
def test_run_host_fused(bits):
    m = bits // 32
    n = max(3, (1 << 26) // bits)
    a, b = inputs.make_operands(n, m, seed=8, cls="MIX")
    a, b = a.pin_memory(), b.pin_memory()
    outs = bn.run_host(["add6", "poly_classical", "poly_ntt"], a, b)
    da, db = a.to(DEV), b.to(DEV)
    assert torch.equal(outs[0], bn.add6(da, db).cpu())
    wp = bn.poly_ntt(da, db).cpu()
    assert torch.equal(outs[1], wp) and torch.equal(outs[2], wp)
    idx = [0, n // 2, n - 1]
    assert np.array_equal(inputs.to_numpy_u32(outs[2][idx]),
                          O.poly(inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx])))


# ------------------------------------------- full (wide) products (§8(f) #2)

@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "MIX"])
@pytest.mark.parametrize("bits", SIZES)
def test_parity_wide(bits, cls):
    """Full 2m-limb products vs the oracle's untruncated schoolbook product,
    bit-exact (NTT: inputs up to 128K bits)."""
    m = bits // 32
    n = max(2, N_INST[bits] // 4) if bits >= 65536 else N_INST[bits]
    a, b = inputs.make_operands(n, m, seed=7 * bits + len(cls), cls=cls)
    want = O.mul_full_rows(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b))
    da, db = a.to(DEV), b.to(DEV)
    got = inputs.to_numpy_u32(bn.mul_wide_classical(da, db))
    bad = _first_bad(got, want)
    assert bad is None, "wide classical %d bits %s: %s" % (bits, cls, bad)
    got = inputs.to_numpy_u32(bn.mul_wide_ntt(da, db))
    bad = _first_bad(got, want)
    assert bad is None, "wide ntt %d bits %s: %s" % (bits, cls, bad)


@pytest.mark.parametrize("cap", [1, 4])
@pytest.mark.parametrize("bits", [1024, 16384])
def test_wide_grid_cap_and_u64(bits, cap):
    m = bits // 32
    a, b = inputs.make_operands(77, m, seed=cap, cls="MIX")
    want = O.mul_full_rows(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b))
    da, db = a.to(DEV), b.to(DEV)
    bn.debug_set_grid_cap(cap)
    try:
        for f in (bn.mul_wide_classical, bn.mul_wide_ntt):
            assert np.array_equal(inputs.to_numpy_u32(f(da, db)), want), f.__name__
            got = f(da.view(torch.int64), db.view(torch.int64)).view(torch.int32)
            assert np.array_equal(inputs.to_numpy_u32(got), want), f.__name__ + " u64"
    finally:
        bn.debug_set_grid_cap(0)
    # out (2m limbs per instance) may not overlap an input: the C ABI
    # rejects it before any launch
    lib = bn.load()
    big = torch.empty((77, 3 * m), dtype=torch.int32, device=DEV)
    st = lib.bn_mul_wide_classical(big.data_ptr(), big.data_ptr(), db.data_ptr(), 77, m, 32, None)
    assert st == 4  # BN_EALIAS
    st = lib.bn_mul_wide_ntt(big.data_ptr(), da.data_ptr(), big.data_ptr(), 77, m, 32, None)
    assert st == 4


def test_wide_full_size_4096():
    """Bench-size batch: classical wide == NTT wide on all 2^20 instances, the
    low half equals the truncated product, and sampled instances match the
    oracle's full product."""
    m, n = 128, 1 << 20
    a, b = inputs.make_operands(n, m, seed=3, cls="U", device=DEV)
    wc = bn.mul_wide_classical(a, b)
    wn = bn.mul_wide_ntt(a, b)
    assert torch.equal(wc, wn)
    assert torch.equal(wc[:, :m], bn.mul_ntt(a, b))
    idx = torch.tensor([0, 12345, n - 1], device=DEV)
    want = O.mul_full_rows(inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx]))
    assert np.array_equal(inputs.to_numpy_u32(wc[idx]), want)


# ------------------------- beyond one CTA: thread-block clusters (§8(f) #4)

CLUSTER_SIZES = [1 << 19, 1 << 20]


@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "RUNS", "MIX"])
@pytest.mark.parametrize("bits", CLUSTER_SIZES)
def test_parity_cluster_sizes(bits, cls):
    """bn_add and bn_mul_ntt at 512K / 1M bits (one instance per cluster of
    2 / 4 CTAs) vs the oracle, bit-exact; carries cross CTA boundaries
    (RIPPLE: through every thread, warp and CTA)."""
    m = bits // 32
    n = 3
    a, b = inputs.make_operands(n, m, seed=bits % 1000 + len(cls), cls=cls)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    got = inputs.to_numpy_u32(bn.add(da, db))
    bad = _first_bad(got, O.add(an, bnp))
    assert bad is None, "add %d %s: %s" % (bits, cls, bad)
    wm = O.mul(an, bnp, nthreads=8)
    got = inputs.to_numpy_u32(bn.mul_ntt(da, db))
    bad = _first_bad(got, wm)
    assert bad is None, "mul_ntt %d %s: %s" % (bits, cls, bad)
    if bits <= bn.max_bits("mul_classical"):
        got = inputs.to_numpy_u32(bn.mul_classical(da, db))
        bad = _first_bad(got, wm)
        assert bad is None, "mul_classical %d %s: %s" % (bits, cls, bad)
    else:
        with pytest.raises(bn.BnError):
            bn.mul_classical(da, db)


@pytest.mark.parametrize("bits", CLUSTER_SIZES)
def test_cluster_full_batch_closed_forms(bits):
    """Paper batch (2^32 bits per operand) at 512K / 1M bits: all-ones closed
    forms on every instance, grid-stride over clusters."""
    m = bits // 32
    n = (1 << 32) // bits
    ones, _ = inputs.make_operands(n, m, seed=1, cls="ONES", device=DEV)
    _, rip = inputs.make_operands(n, m, seed=1, cls="RIPPLE", device=DEV)
    one = torch.zeros((m,), dtype=torch.int32, device=DEV)
    one[0] = 1
    assert torch.equal(bn.mul_ntt(ones, ones), one.expand(n, m))
    assert not bn.add(ones, rip).any()
    assert torch.equal(bn.mul_ntt(ones, rip), ones)
    s = bn.add(ones, ones)
    want = torch.full((m,), -1, dtype=torch.int32, device=DEV)
    want[0] = -2
    assert torch.equal(s, want.expand(n, m))


@pytest.mark.parametrize("cap", [2, 4])
def test_cluster_grid_cap(cap):
    """Clusters that each run several instances (cluster-count cap) give the
    same results as the oracle (R20); exercises the double-buffered CTA
    aggregates of the cluster carry scan."""
    bits = 1 << 19
    m = bits // 32
    a, b = inputs.make_operands(7, m, seed=cap, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    bn.debug_set_grid_cap(cap)
    try:
        ga = inputs.to_numpy_u32(bn.add(da, db))
        gm = inputs.to_numpy_u32(bn.mul_ntt(da, db))
        gc = inputs.to_numpy_u32(bn.mul_classical(da, db))
    finally:
        bn.debug_set_grid_cap(0)
    wm = O.mul(an, bnp, nthreads=8)
    assert _first_bad(ga, O.add(an, bnp)) is None
    assert _first_bad(gm, wm) is None
    assert _first_bad(gc, wm) is None


@pytest.mark.parametrize("bits", CLUSTER_SIZES)
def test_in_place_cluster_sizes(bits):
    """out == a, out == b and a == b == out at the cluster sizes (one
    instance per 2 / 4-CTA cluster): every CTA reads its slice before the
    cluster scan and writes it after (include/bn.h ALIASING AND ORDER)."""
    m = bits // 32
    a, b = inputs.make_operands(3, m, seed=5, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    ops = [("add", bn.add, O.add), ("mul_ntt", bn.mul_ntt, O.mul)]
    if bits <= bn.max_bits("mul_classical"):
        ops.append(("mul_classical", bn.mul_classical, O.mul))
    for name, f, ref in ops:
        da, db = a.to(DEV), b.to(DEV)
        f(da, db, out=da)
        assert np.array_equal(inputs.to_numpy_u32(da), ref(an, bnp)), name + " out=a"
        da = a.to(DEV)
        f(da, db, out=db)
        assert np.array_equal(inputs.to_numpy_u32(db), ref(an, bnp)), name + " out=b"
        da = a.to(DEV)
        f(da, da, out=da)
        assert np.array_equal(inputs.to_numpy_u32(da), ref(an, an)), name + " a=b=out"


@pytest.mark.parametrize("bits", [4096, 32768, 262144])
def test_in_place_fused(bits):
    """6-Add and Poly (both multiplications) in place at 4K bits and above:
    out == a, out == b, a == b == out."""
    m = bits // 32
    n = {4096: 37, 32768: 5, 262144: 2}[bits]
    a, b = inputs.make_operands(n, m, seed=11, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    ops = [("add6", lambda x, y, out: bn.add6(x, y, out=out), O.add6)]
    for name in ("poly_classical", "poly_ntt"):
        f = getattr(bn, name)
        ops.append((name, lambda x, y, out, f=f: f(x, y, out=out), O.poly))
    for name, f, ref in ops:
        da, db = a.to(DEV), b.to(DEV)
        f(da, db, out=da)
        assert np.array_equal(inputs.to_numpy_u32(da), ref(an, bnp)), name + " out=a"
        da = a.to(DEV)
        f(da, db, out=db)
        assert np.array_equal(inputs.to_numpy_u32(db), ref(an, bnp)), name + " out=b"
        da = a.to(DEV)
        f(da, da, out=da)
        assert np.array_equal(inputs.to_numpy_u32(da), ref(an, an)), name + " a=b=out"


@pytest.mark.parametrize("bits", [65536, 131072, 262144])
@pytest.mark.parametrize("cap", [1, 3])
def test_add6_prefetch_grid_cap(bits, cap):
    """The TMA-prefetch 6-Add (64K bits and up: one shared stage per
    persistent CTA, refilled with the CTA's next instance after the first
    scan) with CTAs that run several instances (grid cap), ragged n, RIPPLE
    operands (carries through every chunk), and in place (out == a, out == b):
    bit-exact vs the oracle."""
    m = bits // 32
    n = 7
    a, b = inputs.make_operands(n, m, seed=60 + cap, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    r, s = inputs.make_operands(n, m, seed=61, cls="RIPPLE")
    rn, sn = inputs.to_numpy_u32(r), inputs.to_numpy_u32(s)
    bn.debug_set_grid_cap(cap)
    try:
        da, db = a.to(DEV), b.to(DEV)
        assert np.array_equal(inputs.to_numpy_u32(bn.add6(da, db)), O.add6(an, bnp))
        dr, ds = r.to(DEV), s.to(DEV)
        assert np.array_equal(inputs.to_numpy_u32(bn.add6(dr, ds)), O.add6(rn, sn))
        bn.add6(da, db, out=da)
        assert np.array_equal(inputs.to_numpy_u32(da), O.add6(an, bnp)), "out=a"
        da = a.to(DEV)
        bn.add6(da, db, out=db)
        assert np.array_equal(inputs.to_numpy_u32(db), O.add6(an, bnp)), "out=b"
    finally:
        bn.debug_set_grid_cap(0)


@pytest.mark.parametrize("cap", [1, 3])
def test_wide_ntt_256k_grid_cap(cap):
    """The 256K wide NTT kernel (one 512-thread CTA per instance, incremental
    Garner) with CTAs that run several instances (grid cap): bit-exact vs the
    oracle's full product and the classical wide kernel."""
    bits = 262144
    m = bits // 32
    a, b = inputs.make_operands(5, m, seed=40 + cap, cls="MIX")
    want = O.mul_full_rows(inputs.to_numpy_u32(a), inputs.to_numpy_u32(b))
    da, db = a.to(DEV), b.to(DEV)
    bn.debug_set_grid_cap(cap)
    try:
        got = inputs.to_numpy_u32(bn.mul_wide_ntt(da, db))
    finally:
        bn.debug_set_grid_cap(0)
    assert _first_bad(got, want) is None
    ones, _ = inputs.make_operands(3, m, seed=1, cls="ONES", device=DEV)
    w = bn.mul_wide_ntt(ones, ones)  # (2^B - 1)^2 = 2^2B - 2^(B+1) + 1
    exp = torch.zeros((2 * m,), dtype=torch.int32, device=DEV)
    exp[0] = 1
    exp[m] = -2
    exp[m + 1:] = -1
    assert torch.equal(w, exp.expand(3, 2 * m))


# ------------------------- beyond clusters: decoupled look-back (§8(f) #4)

@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "RUNS", "MIX"])
@pytest.mark.parametrize("bits", [1 << 18, 1 << 20, 1 << 21, 1 << 23])
def test_parity_add_big(bits, cls):
    """bn_add_big (tiles of 2^18 bits, decoupled look-back carry scan) vs the
    oracle, bit-exact: RIPPLE carries through every tile of an instance, ONES
    makes every tile all-propagate (the look-back walks back to a decisive
    tile); at 2^18 .. 2^20 also equal to bn_add (one CTA / cluster)."""
    m = bits // 32
    n = 5 if bits <= (1 << 21) else 2
    a, b = inputs.make_operands(n, m, seed=bits % 977 + len(cls), cls=cls)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    da, db = a.to(DEV), b.to(DEV)
    got = bn.add_big(da, db)
    bad = _first_bad(inputs.to_numpy_u32(got), O.add(an, bnp))
    assert bad is None, "add_big %d %s: %s" % (bits, cls, bad)
    if bits <= bn.max_bits("add"):
        assert torch.equal(got, bn.add(da, db))


def test_add_big_worst_case_chain_and_in_place():
    """2^26-bit instances (256 tiles each), a = 2^B - 1, b = 1: one carry
    through every limb of every tile; in place (out == a) too; and a batch
    whose instance boundaries cut the look-back (instance k's first tile must
    not take instance k-1's carry, reading R1)."""
    bits = 1 << 26
    m = bits // 32
    ones, _ = inputs.make_operands(3, m, seed=1, cls="ONES", device=DEV)
    one = torch.zeros((3, m), dtype=torch.int32, device=DEV)
    one[:, 0] = 1
    assert not bn.add_big(ones, one).any()               # (2^B - 1) + 1 = 0 mod 2^B, every instance
    s = bn.add_big(ones, ones, out=ones)                  # in place: 2^(B+1) - 2 mod 2^B
    want = torch.full((m,), -1, dtype=torch.int32, device=DEV)
    want[0] = -2
    assert torch.equal(s, want.expand(3, m))


@pytest.mark.parametrize("bits", [1 << 22])
def test_add_big_u64_and_paper_batch(bits):
    """u64 limbs are the same bytes; the paper batch (2^32 bits per operand)
    sampled against the oracle."""
    m = bits // 32
    n = (1 << 32) // bits
    a, b = inputs.make_operands(n, m, seed=9, cls="MIX", device=DEV)
    r32 = bn.add_big(a, b)
    r64 = bn.add_big(a.view(torch.int64), b.view(torch.int64)).view(torch.int32)
    assert torch.equal(r32, r64)
    idx = torch.tensor([0, n // 2, n - 1], device=DEV)
    want = O.add(inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx]))
    assert np.array_equal(inputs.to_numpy_u32(r32[idx]), want)
