"""CPU model of the NTT kernel's data layout (mul_ntt.cu) — -m "not gpu".

Checks the index algebra the kernel relies on, for every N = 2^6 .. 2^14:
* pass p's 16 register elements of thread t are indices whose bits
  [LO_p, LO_p + 4) vary, and every forward stage s of the pass pairs elements
  held by the same thread (butterfly partner u ^ 2^(N-1-s));
* the per-stage twiddle index (u mod 2^beta) is tlow + (e_low << LO);
* the XOR swizzle swz(u) = u ^ (r ^ (r << 1)), r = (u >> 5) & 15, is a
  bijection on [0, N) and every warp access of every pass is
  bank-conflict-free (32 distinct banks per 4-byte access);
* the L/H publish of the CRT epilogue (Q = 8 consecutive coefficients per
  thread) never writes one H slot twice and covers every slot.
"""
import pytest

R_LOG = 4


def passes(logn):
    np_ = (logn + 3) // 4
    out = []
    for p in range(np_):
        s0 = 4 * p
        s1 = min(4 * p + 4, logn)
        lo = max(logn - 4 * (p + 1), 0)
        out.append((s0, s1, lo))
    return out


def lay(t, e, lo):
    return (t & ((1 << lo) - 1)) | (e << lo) | ((t >> lo) << (lo + 4))


def swz(u):
    r = (u >> 5) & 15
    return u ^ (r ^ (r << 1))


def xaddr(logn, u):
    """the kernel's physical word of CTA-wide index u (mul_ntt.cu xbase/xaddr)."""
    return u + (u >> 4) if logn <= 8 else swz(u)


def xaddr_split(logn, lo, T, e):
    """the kernel's split form: thread base combined with the compile-time e part."""
    E = e << lo
    if logn <= 8:
        base = T + (T >> 4)
        return base + E + (E >> 4)
    base = swz(T)
    hE = swz(E) ^ E
    if lo >= 5:
        return (base ^ hE) + E
    return (base ^ ((E & 31) ^ hE)) + (E & ~31)


@pytest.mark.parametrize("logn", range(6, 15))
def test_pass_groups_and_twiddle_index(logn):
    N = 1 << logn
    tpi = N >> R_LOG
    for (s0, s1, lo) in passes(logn):
        seen = set()
        for t in range(tpi):
            us = [lay(t, e, lo) for e in range(16)]
            seen.update(us)
            for s in range(s0, s1):
                beta = logn - 1 - s
                b = beta - lo
                assert 0 <= b < 4
                for e in range(16):
                    if e & (1 << b):
                        continue
                    u, v = us[e], us[e | (1 << b)]
                    assert v == u + (1 << beta)                  # DIF partner
                    j = u & ((1 << beta) - 1)                     # twiddle exponent / 2^s
                    tlow = t & ((1 << lo) - 1)
                    assert j == tlow + ((e & ((1 << b) - 1)) << lo)
        assert seen == set(range(N))                              # a partition of [0, N)


@pytest.mark.parametrize("logn", range(6, 15))
def test_exchange_addressing_bijective_and_conflict_free(logn):
    N = 1 << logn
    tpi = N >> R_LOG
    ipb = 1 if tpi >= 256 else 256 // tpi
    span = ipb * N
    phys = [xaddr(logn, u) for u in range(span)]
    assert len(set(phys)) == span                                 # injective
    xw = span + (span >> 4) if logn <= 8 else span
    assert max(phys) < xw                                         # fits the XW words
    for (_, _, lo) in passes(logn):
        for w0 in range(0, min(ipb * tpi, 256), 32):
            lanes = range(w0, w0 + 32)
            for e in range(16):
                addrs = []
                for t in lanes:
                    slot, tt = t // tpi, t % tpi
                    u = slot * N + lay(tt, e, lo)
                    T = slot * N + ((tt & ((1 << lo) - 1)) | ((tt >> lo) << (lo + 4)))
                    a = xaddr(logn, u)
                    assert xaddr_split(logn, lo, T, e) == a              # split form is exact
                    addrs.append(a)
                assert len({a % 32 for a in addrs}) == 32, (logn, lo, e)  # no bank conflict


@pytest.mark.parametrize("logn", range(6, 15))
def test_epilogue_publish_layout(logn):
    M = 1 << (logn - 1)
    tpi = (1 << logn) >> R_LOG
    Q = M // tpi
    assert Q == 8
    writes = {}
    for t in range(tpi):
        for q in range(Q):
            base = Q * t + Q if Q * t + Q < M else 0
            slot = base + q
            assert slot not in writes
            writes[slot] = t
    assert set(writes) == set(range(M))


@pytest.mark.parametrize("logn", range(6, 15))
def test_slot_regions_disjoint(logn):
    """Each instance slot's exchange addresses stay inside its own region of
    XW / IPB words, which is also where L | H are published: slots in
    different warps synchronise only at CTA barriers (mul_ntt.cu, the race
    fixed after the full-size 4096-bit parity run)."""
    N = 1 << logn
    tpi = N >> R_LOG
    ipb = 1 if tpi >= 256 else 256 // tpi
    xw = ipb * N + (ipb * N >> 4) if logn <= 8 else ipb * N
    region = xw // ipb
    assert region >= N  # room for L | H (N = 2m words)
    for slot in range(ipb):
        for u in range(N):
            a = xaddr(logn, slot * N + u)
            assert slot * region <= a < (slot + 1) * region


def cswz(q, k):
    """mul_ntt.cu cswz<Q>: XOR the 16-byte chunk index inside each 32-word row
    with the row number's low bits."""
    return k ^ (((k >> 5) & (q // 4 - 1)) << 2)


def _wavefronts_128(addrs):
    """Shared-memory wavefronts of one quarter-warp's 128-bit accesses: the
    number of distinct 16-byte chunks that fall in the same bank group."""
    groups = {}
    for a in addrs:
        groups.setdefault((a // 4) % 8, set()).add(a // 4)
    return max(len(v) for v in groups.values())


@pytest.mark.parametrize("q", [8, 16])
@pytest.mark.parametrize("logm", range(5, 14))
def test_epilogue_swizzle_conflict_free(q, logm):
    """cswz<Q> is a bijection on [0, M) that keeps 16-byte chunks whole; a
    warp's pass-layout writes (32 consecutive words, or two aligned 16-word
    halves) stay conflict free; every quarter-warp's Q-words-per-thread
    128-bit access (owners t .. t+7, also shifted by one owner as the H
    publish is) hits 8 distinct bank groups — where plain row-major needs
    Q/4 wavefronts."""
    M = 1 << logm
    perm = [cswz(q, k) for k in range(M)]
    assert sorted(perm) == list(range(M))
    assert all(cswz(q, k) // 4 == cswz(q, k - k % 4) // 4 and cswz(q, k) % 4 == k % 4 for k in range(M))
    # pass-layout writes: aligned runs of 16 consecutive words map onto one aligned 16-word group
    for k0 in range(0, M, 16):
        banks = {cswz(q, k) % 32 for k in range(k0, k0 + 16)}
        assert len(banks) == 16 and len({b // 16 for b in banks}) == 1
    owners = M // q
    for shift in (0, 1):
        for t0 in range(0, owners - 8 - shift + 1, 8):
            for c in range(q // 4):
                addrs = [cswz(q, (t + shift) * q + 4 * c) for t in range(t0, t0 + 8)]
                assert _wavefronts_128(addrs) == 1
                plain = [(t + shift) * q + 4 * c for t in range(t0, t0 + 8)]
                if owners >= 8:
                    assert _wavefronts_128(plain) == q // 4
