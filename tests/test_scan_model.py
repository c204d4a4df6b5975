"""CPU model of the carry-scan algebra the add kernel uses — -m "not gpu".

Pins the paper's operators (Figs. 2/3) and the warp-level
ballot-add formulation used in csrc/bn_scan.cuh against sequential folds:

* carry_op_nice / carry_op_eff /
  carry_op_sgm: associativity, identity, eff == nice.
* ballot-add: with G = generate mask, P = propagate mask, X = G|P,
  carry-in mask = (X + G + c0) ^ X ^ G equals the exclusive scan of
  carry_op_eff over lanes (all 3^8 patterns of 8 lanes + random 32-lane).
* segment isolation (reading R1): clearing the (g, p) bits of the top lane of
  every segment gives each segment carry-in 0, whereas the literal exclusive
  segmented scan leaks the previous segment's carry.
"""
import itertools

import pytest
import random


def carry_op_nice(x, y):
    ov1, mx1 = x
    ov2, mx2 = y
    return ((ov1 and mx2) or ov2, mx1 and mx2)


def carry_op_eff(c1, c2):
    return (c1 & c2 & 2) | (((c1 & (c2 >> 1)) | c2) & 1)


def carry_op_sgm(c1, c2):
    if c2 & 4:
        return c2
    return carry_op_eff(c1, c2) | ((c1 | c2) & 4)


def test_eff_equals_nice_and_identity():
    for ov1, mx1, ov2, mx2 in itertools.product((0, 1), repeat=4):
        n = carry_op_nice((bool(ov1), bool(mx1)), (bool(ov2), bool(mx2)))
        e = carry_op_eff(ov1 | (mx1 << 1), ov2 | (mx2 << 1))
        assert e == int(n[0]) | (int(n[1]) << 1)
    for c in range(4):
        assert carry_op_eff(2, c) == c and carry_op_eff(c, 2) == c
    for c in range(8):
        assert carry_op_sgm(2, c) == c or (c & 4)  # 2 is neutral up to the segment bit


def test_associativity_exhaustive():
    for a, b, c in itertools.product(range(4), repeat=3):
        assert carry_op_eff(carry_op_eff(a, b), c) == carry_op_eff(a, carry_op_eff(b, c))
    for a, b, c in itertools.product(range(8), repeat=3):
        assert carry_op_sgm(carry_op_sgm(a, b), c) == carry_op_sgm(a, carry_op_sgm(b, c))


def _excl_scan(op, e, xs):
    out, acc = [], e
    for x in xs:
        out.append(acc)
        acc = op(acc, x)
    return out


def _ballot_cin(gs, ps, c0, width):
    """the kernel's formula: carry-in mask = (X + G + c0) ^ X ^ G, X = G|P."""
    G = sum(g << i for i, g in enumerate(gs))
    P = sum(p << i for i, p in enumerate(ps))
    X = G | P
    S = X + G + c0
    cin = (S ^ X ^ G) & ((1 << width) - 1)
    cout = (S >> width) & 1
    return [(cin >> i) & 1 for i in range(width)], cout


def _seq(gs, ps, c0):
    cins, c = [], c0
    for g, p in zip(gs, ps):
        cins.append(c)
        c = g | (p & c)
    return cins, c


def test_ballot_add_all_8_lane_patterns():
    # kill / generate / propagate per lane (g and p exclusive, as for chunk sums)
    for pat in itertools.product((0, 1, 2), repeat=8):
        gs = [int(x == 1) for x in pat]
        ps = [int(x == 2) for x in pat]
        for c0 in (0, 1):
            assert _ballot_cin(gs, ps, c0, 8) == _seq(gs, ps, c0)
            # and equals the paper's exclusive scan of carry_op_eff (ov=g, mx=p)
            if c0 == 0:
                sc = _excl_scan(carry_op_eff, 2, [g | (p << 1) for g, p in zip(gs, ps)])
                assert [s & 1 for s in sc] == _seq(gs, ps, 0)[0]


def test_ballot_add_random_32_lane():
    rng = random.Random(5)
    for _ in range(20000):
        pat = [rng.choice((0, 1, 2, 2, 2)) for _ in range(32)]
        gs = [int(x == 1) for x in pat]
        ps = [int(x == 2) for x in pat]
        c0 = rng.randrange(2)
        assert _ballot_cin(gs, ps, c0, 32) == _seq(gs, ps, c0)


def test_segment_isolation():
    """IPB = 4 segments of 8 lanes: top lane of each segment masked to kill."""
    rng = random.Random(9)
    seg = 8
    for _ in range(5000):
        pat = [rng.choice((0, 1, 2)) for _ in range(32)]
        gs = [int(x == 1) for x in pat]
        ps = [int(x == 2) for x in pat]
        mg = [0 if i % seg == seg - 1 else g for i, g in enumerate(gs)]
        mp = [0 if i % seg == seg - 1 else p for i, p in enumerate(ps)]
        cins, _ = _ballot_cin(mg, mp, 0, 32)
        for s in range(0, 32, seg):
            want, _ = _seq(gs[s:s + seg], ps[s:s + seg], 0)
            assert cins[s:s + seg] == want


def test_literal_segmented_scan_leaks():
    """Reading R1: Fig. 2's scan^exc carry_op_sgm 2 with the segment bit on
    the head element passes the previous segment's carry into the head."""
    # two instances of M=2 limbs: (all-ones + 1) then (0 + 0)
    M, MAX = 2, 0xFFFFFFFF
    a = [MAX, MAX, 0, 0]
    b = [1, 0, 0, 0]
    flags = []
    for i, (x, y) in enumerate(zip(a, b)):
        p = (x + y) & MAX
        flags.append((4 if i % M == 0 else 0) | ((p == MAX) << 1) | int(p < x))
    carries = _excl_scan(carry_op_sgm, 2, flags)
    assert carries[2] & 1 == 1  # the carry of instance 0 leaks into instance 1


def _model_add(xs, ys, L, TPI):
    """Python model of csrc/bn_common.cuh add_regs over one instance:
    chunk_sum -> ballot-add carry scan across TPI threads -> chunk_apply."""
    MAX = 0xFFFFFFFF
    gs, ps, sums = [], [], []
    for t in range(TPI):
        x, y = xs[t * L:(t + 1) * L], ys[t * L:(t + 1) * L]
        s = [(a + b) & MAX for a, b in zip(x, y)]
        g, p = 0, 1
        for a, v in zip(x, s):
            ov, mx = int(v < a), int(v == MAX)
            g = ov | (mx & g)
            p &= mx
        gs.append(g)
        ps.append(p)
        sums.append(s)
    cins, _ = _ballot_cin(gs, ps, 0, TPI)
    out = []
    for t in range(TPI):
        x, s, c = xs[t * L:(t + 1) * L], sums[t], cins[t]
        for a, v in zip(x, s):
            out.append((v + c) & MAX)
            c = int(v < a) | (int(v == MAX) & c)
    return out


def test_model_add_matches_python_int():
    rng = random.Random(11)
    for L, TPI in ((8, 4), (8, 32), (4, 16), (16, 8)):
        M = L * TPI
        for trial in range(300):
            kind = trial % 4
            if kind == 0:
                xs = [rng.getrandbits(32) for _ in range(M)]
                ys = [rng.getrandbits(32) for _ in range(M)]
            elif kind == 1:
                xs, ys = [0xFFFFFFFF] * M, [1] + [0] * (M - 1)
            elif kind == 2:
                xs = [rng.getrandbits(32) for _ in range(M)]
                ys = [(~v + (rng.random() < 0.05)) & 0xFFFFFFFF for v in xs]
            else:
                xs, ys = [0xFFFFFFFF] * M, [0xFFFFFFFF] * M
            A = sum(v << (32 * i) for i, v in enumerate(xs))
            B = sum(v << (32 * i) for i, v in enumerate(ys))
            S = (A + B) % (1 << (32 * M))
            assert _model_add(xs, ys, L, TPI) == [(S >> (32 * i)) & 0xFFFFFFFF for i in range(M)]


def _chunk_sum(x, y, cin, L):
    """bn_common.cuh chunk_sum on one L-limb chunk with carry-in cin: (s, g, p)."""
    mask = (1 << (32 * L)) - 1
    t = x + y + cin
    s = t & mask
    return s, t >> (32 * L), int(s == mask)


def _scan_exclusive(gs, ps):
    """exclusive carry scan over chunks (carry_op of PAPER.md:177-215)."""
    out, c = [], 0
    for g, p in zip(gs, ps):
        out.append(c)
        c = g | (p & c)
    return out


def _six_add_carry_save(a, b, n_chunks, L):
    """Model of add6_kernel with BN_ADD6_CS (bn_common.cuh add_pending): the
    final increment of addition k rides in addition k+1's carry chain, with
    the carry-out cleared when the pending chunk was all ones with carry-in 1."""
    W = 32 * L
    mask = (1 << W) - 1
    ca = [(a >> (W * j)) & mask for j in range(n_chunks)]
    cb = [(b >> (W * j)) & mask for j in range(n_chunks)]
    s, g, p = zip(*[_chunk_sum(x, y, 0, L) for x, y in zip(ca, cb)])
    s, p = list(s), list(p)
    cin = _scan_exclusive(g, p)
    for k in range(1, 6):
        z = ca if k % 2 else cb
        gs = []
        for j in range(n_chunks):
            ov = p[j] & cin[j]
            s[j], gj, p[j] = _chunk_sum(s[j], z[j], cin[j], L)
            gs.append(gj & (1 - ov))
        cin = _scan_exclusive(gs, p)
    r = [(s[j] + cin[j]) & mask for j in range(n_chunks)]
    return sum(v << (W * j) for j, v in enumerate(r))


@pytest.mark.parametrize("L,n_chunks", [(1, 8), (2, 5), (4, 3)])
def test_six_add_carry_save_model(L, n_chunks):
    """The carry-save 6-Add equals six sequential additions (4a + 3b mod 2^B,
    reading R17) on random, all-ones and carry-run inputs — in particular the
    double-count case (pending chunk all ones with carry-in 1)."""
    import random
    rng = random.Random(L * 100 + n_chunks)
    B = 32 * L * n_chunks
    mod = 1 << B
    ones = mod - 1
    cases = [(ones, ones), (ones, 1), (1, ones), (0, ones), (ones, 0), (ones >> 1, ones)]
    for _ in range(3000):
        kind = rng.randrange(4)
        if kind == 0:
            a, b = rng.getrandbits(B), rng.getrandbits(B)
        elif kind == 1:  # long runs of ones with sparse holes
            a = ones ^ (1 << rng.randrange(B)) if rng.random() < 0.7 else ones
            b = rng.getrandbits(8) << rng.randrange(B - 8)
        elif kind == 2:  # chunks that are all ones / zero
            W = 32 * L
            a = sum(rng.choice([0, (1 << W) - 1, rng.getrandbits(W)]) << (W * j) for j in range(n_chunks))
            b = sum(rng.choice([0, 1, (1 << W) - 1]) << (W * j) for j in range(n_chunks))
        else:  # b = ~a + small -> 3b + 4a lands near multiples of 2^W
            a = rng.getrandbits(B)
            b = (ones ^ a) + rng.randrange(3)
        cases.append((a % mod, b % mod))
    for a, b in cases:
        want = a
        want = (a + b) % mod
        for k in range(1, 6):
            want = (want + (a if k % 2 else b)) % mod
        assert _six_add_carry_save(a, b, n_chunks, L) == want, (hex(a), hex(b))


def _lookback_carry(tile, lt, flags):
    """Model of add_lookback_kernel's warp-wide look-back (add.cu): window of
    32 predecessors, lane k reads tile - 1 - k (lanes at or past the
    instance's first tile are decisive with carry 0); a predecessor is
    decisive if its inclusive carry is published (status 2) or its aggregate
    does not propagate (p = 0, carry = g); the nearest decisive one wins."""
    base, remaining = tile, lt
    while True:
        lanes = []
        for k in range(32):
            if k < remaining:
                st, g, p, inc = flags[base - 1 - k]
                assert st != 0, "the kernel spins until a flag is published"
                dec = st == 2 or p == 0
                lanes.append((dec, (inc if st == 2 else g)))
            else:
                lanes.append((True, 0))
        ds = [k for k, (d, _) in enumerate(lanes) if d]
        if ds:
            return lanes[ds[0]][1] if ds[0] < remaining else 0
        base -= 32
        remaining -= 32


@pytest.mark.parametrize("tiles_per_inst", [1, 5, 33, 70])
def test_decoupled_lookback_model(tiles_per_inst):
    """The look-back decision equals the sequential carry into every tile
    (carry_op of PAPER.md:177-215 folded from the instance's first tile), for
    tiles that are all-propagate for long stretches (> 32, so the window
    slides) and any mix of published aggregate / inclusive flags; carries
    never cross an instance boundary (reading R1)."""
    import random
    rng = random.Random(tiles_per_inst)
    n_inst = 3
    for trial in range(200):
        aggs = []
        for i in range(n_inst * tiles_per_inst):
            r = rng.random()
            if trial % 3 == 0:
                g, p = (0, 1) if rng.random() < 0.95 else (rng.randrange(2), 0)  # long propagate runs
            else:
                g, p = (1, 0) if r < 0.3 else (0, 0) if r < 0.6 else (0, 1)
            aggs.append((g, p))
        # true carries: fold within each instance
        true_cin, incl = [], []
        for i, (g, p) in enumerate(aggs):
            c = 0 if i % tiles_per_inst == 0 else incl[-1]
            true_cin.append(c)
            incl.append(g | (p & c))
        # every tile's aggregate is published; a random subset also has its inclusive flag
        flags = [(2 if rng.random() < 0.5 else 1, g, p, incl[i]) for i, (g, p) in enumerate(aggs)]
        for t in range(len(aggs)):
            lt = t % tiles_per_inst
            got = 0 if lt == 0 else _lookback_carry(t, lt, flags)
            assert got == true_cin[t], (trial, t)
