"""Python models of the two multiplication kernels' algorithms — -m "not gpu".

These re-execute, in exact integer arithmetic with explicit 32-bit wrap-
around, the per-thread work decomposition of csrc/mul_classical.cu (mirrored
Q-column chunks, sliding B window with a zero chunk in front, 96-bit column
accumulators, `combine`, L/H publish, R = L + H) and csrc/mul_ntt.cu (lazy
DIF/DIT passes with Shoup twiddles, Montgomery pointwise, Garner CRT with the
folded 2^32 N^-1 constants, 8-coefficient aggregates, L/H publish), and
compare against Python-int products.  They validate the index algebra and the
lazy-reduction bounds on the CPU before any GPU run; the GPU parity tests
validate the kernels themselves.
"""
import random

import pytest

MASK = 0xFFFFFFFF


def to_int(limbs):
    return sum(v << (32 * i) for i, v in enumerate(limbs))


def from_int(v, m):
    return [(v >> (32 * i)) & MASK for i in range(m)]


# ------------------------------------------------------------------ classical

def model_classical(A, B, Q):
    m = len(A)
    G = m // (2 * Q)
    Bz = [0] * Q + B                     # B[-Q..-1] = 0 (zero chunk)

    def Bx(x):
        return Bz[x + Q]

    def conv_chunk(j0):
        lo, hi, top = [0] * Q, [0] * Q, [0] * Q
        cur = [Bx(Q * j0 + q) for q in range(Q)]
        for c in range(j0 + 1):
            av = A[Q * c:Q * c + Q]
            prev = [Bx(Q * (j0 - c - 1) + q) for q in range(Q)]
            for s in range(Q):
                for q in range(Q):
                    d = q - s
                    bj = cur[d] if d >= 0 else prev[Q + d]
                    acc = lo[q] + (hi[q] << 32) + (top[q] << 64) + av[s] * bj
                    lo[q], hi[q], top[q] = acc & MASK, (acc >> 32) & MASK, (acc >> 64) & MASK
            cur = prev
        # combine
        lh = [0] * (Q + 2)
        lh[0] = lo[0]
        h_res, c_res = hi[0], top[0]
        for q in range(1, Q):
            l, h = lo[q], hi[q]
            lh[q] = (l + h_res) & MASK
            h_res = (h + c_res + int(lh[q] < l)) & MASK
            c_res = (top[q] + int(h_res < h)) & MASK
        lh[Q], lh[Q + 1] = h_res, c_res
        return lh

    L, H = [None] * m, [None] * m
    for g in range(G):
        for j0 in (g, m // Q - 1 - g):
            lh = conv_chunk(j0)
            k1 = Q * j0
            for q in range(Q):
                L[k1 + q] = lh[q]
            hs = [lh[Q], lh[Q + 1]] + [0] * (Q - 2)
            base = k1 + Q if k1 + Q < m else 0
            for q in range(Q):
                assert base + q < m
                H[base + q] = hs[q] if base else 0
    assert None not in L and None not in H
    return from_int((to_int(L) + to_int(H)) % (1 << (32 * m)), m)


@pytest.mark.parametrize("m,Q", [(32, 4), (64, 4), (128, 4), (256, 8), (64, 8)])
def test_classical_model(m, Q):
    rng = random.Random(m * Q)
    cases = [([MASK] * m, [MASK] * m), ([MASK] * m, [1] + [0] * (m - 1))]
    cases += [([rng.getrandbits(32) for _ in range(m)], [rng.getrandbits(32) for _ in range(m)])
              for _ in range(4)]
    for A, B in cases:
        want = from_int(to_int(A) * to_int(B) % (1 << (32 * m)), m)
        assert model_classical(A, B, Q) == want


# ------------------------------------------------------------------------ NTT

PRIMES = [1070727169, 1071513601, 1073479681]  # the library's set (bn_ntt_primes; test_abi checks)


def _prim_root(p):
    n, fs, q = p - 1, [], 2
    while q * q <= n:
        if n % q == 0:
            fs.append(q)
            while n % q == 0:
                n //= q
        q += 1
    if n > 1:
        fs.append(n)
    g = 2
    while any(pow(g, (p - 1) // f, p) == 1 for f in fs):
        g += 1
    return g


def shoup(x, w, p):
    wsh = (w << 32) // p
    q = (x * wsh) >> 32
    r = (x * w - q * p) & MASK
    assert r < 2 * p
    return r


def red2(x, m):
    return min(x, (x - m) & MASK)


def mont(a, b, p):
    pinv = (-pow(p, -1, 1 << 32)) & MASK
    t = a * b
    mm = (t & MASK) * pinv & MASK
    u = (t + mm * p) >> 32
    assert u < 2 * p
    return u


def passes(logn):
    out = []
    for P in range((logn + 3) // 4):
        out.append((4 * P, min(4 * P + 4, logn), max(logn - 4 * (P + 1), 0)))
    return out


def lay(t, e, lo):
    return (t & ((1 << lo) - 1)) | (e << lo) | ((t >> lo) << (lo + 4))


def model_ntt_mul(A, B):
    m = len(A)
    N = 2 * m
    logn = N.bit_length() - 1
    tpi = N // 16
    ps = passes(logn)
    res = []
    for p in PRIMES:
        g = _prim_root(p)
        w = pow(g, (p - 1) // N, p)
        wi = pow(w, p - 2, p)
        p2 = 2 * p

        def tw(base, s, j):
            return pow(base, j << s, p)

        def fwd(vals):
            X = list(vals)  # global index space; values per index
            for (s0, s1, lo) in ps:
                for t in range(tpi):
                    us = [lay(t, e, lo) for e in range(16)]
                    x = [X[u] for u in us]
                    for s in range(s0, s1):
                        b = (logn - 1 - s) - lo
                        for e in range(16):
                            if e & (1 << b):
                                continue
                            j = us[e] & ((1 << (logn - 1 - s)) - 1)
                            u_, v_ = x[e], x[e | (1 << b)]
                            assert u_ < p2 and v_ < p2
                            x[e] = red2((u_ + v_) & MASK, p2)
                            if lo == 0 and (e & ((1 << b) - 1)) == 0:   # w^0: no product
                                assert j == 0
                                x[e | (1 << b)] = red2((u_ - v_ + p2) & MASK, p2)
                            else:
                                x[e | (1 << b)] = shoup((u_ - v_ + p2) & MASK, tw(w, s, j), p)
                    for e in range(16):
                        X[us[e]] = x[e]
            return X

        def inv(vals):
            X = list(vals)
            for (s0, s1, lo) in reversed(ps):
                for t in range(tpi):
                    us = [lay(t, e, lo) for e in range(16)]
                    x = [X[u] for u in us]
                    for s in range(s1 - 1, s0 - 1, -1):
                        b = (logn - 1 - s) - lo
                        for e in range(16):
                            if e & (1 << b):
                                continue
                            j = us[e] & ((1 << (logn - 1 - s)) - 1)
                            u_ = red2(x[e], p2)
                            if lo == 0 and (e & ((1 << b) - 1)) == 0:   # w^0: no product
                                assert j == 0
                                v_ = red2(x[e | (1 << b)], p2)
                            else:
                                v_ = shoup(x[e | (1 << b)], tw(wi, s, j), p)
                            x[e] = (u_ + v_) & MASK
                            x[e | (1 << b)] = (u_ - v_ + p2) & MASK
                            assert x[e] < 4 * p and x[e | (1 << b)] < 4 * p
                    for e in range(16):
                        X[us[e]] = x[e]
            return X

        ra = [red2(red2(v, p2), p2) for v in A] + [0] * m   # a_i < 2^32 < 6p
        rb = [red2(red2(v, p2), p2) for v in B] + [0] * m
        assert max(ra + rb) < p2
        fa, fb = fwd(ra), fwd(rb)
        prod = [mont(x, y, p) for x, y in zip(fa, fb)]
        res.append(inv(prod)[:m])
    # Garner with folded constants (bn_api.cu build_tables)
    p0, p1, p2_ = PRIMES
    K = [(pow(2, 32, p) * pow(N, p - 2, p)) % p for p in PRIMES]
    i01 = pow(p0, p1 - 2, p1)
    i012 = pow(p0 * p1 % p2_, p2_ - 2, p2_)
    coeffs = []
    for y0, y1, y2 in zip(*res):
        r0 = red2(shoup(y0, K[0], p0), p0)
        u = shoup(y1, K[1] * i01 % p1, p1)
        v = shoup(r0, i01, p1)
        t1 = red2(red2((u + 2 * p1 - v) & MASK, 2 * p1), p1)
        a2 = shoup(y2, K[2] * i012 % p2_, p2_)
        b2 = shoup(r0, i012, p2_)
        c2 = shoup(t1, p0 * i012 % p2_, p2_)
        d = red2((b2 + c2) & MASK, 2 * p2_)
        t2 = red2(red2((a2 + 2 * p2_ - d) & MASK, 2 * p2_), p2_)
        coeffs.append(r0 + p0 * t1 + p0 * p1 * t2)
    # 8-coefficient aggregates, L/H publish, R = L + H
    L, H = [0] * m, [0] * m
    for t in range(tpi):
        S = sum(coeffs[8 * t + q] << (32 * q) for q in range(8))
        lows = [(S >> (32 * q)) & MASK for q in range(8)]
        over = S >> 256
        assert over < 1 << 64
        L[8 * t:8 * t + 8] = lows
        if 8 * t + 8 < m:
            H[8 * t + 8] = over & MASK
            H[8 * t + 9] = over >> 32
    return from_int((to_int(L) + to_int(H)) % (1 << (32 * m)), m)


@pytest.mark.parametrize("m", [32, 64, 128])
def test_ntt_model(m):
    rng = random.Random(m)
    cases = [([MASK] * m, [MASK] * m), ([MASK] * m, [1] + [0] * (m - 1))]
    cases += [([rng.getrandbits(32) for _ in range(m)], [rng.getrandbits(32) for _ in range(m)])
              for _ in range(2)]
    for A, B in cases:
        want = from_int(to_int(A) * to_int(B) % (1 << (32 * m)), m)
        assert model_ntt_mul(A, B) == want


# ---------------------------------------------------------------------------
# Squaring block selection of conv_chunk_sqr (mul_classical.cu, Poly's a*a
# and b*b): for every column chunk j0, the full blocks c < j0//2 plus the
# parity-masked boundary block c = j0//2 must form each pair i < j of the
# column exactly once (doubled) and the diagonal i == j once (single) —
# against the definition sum_{i+j=k} a_i a_j, exhaustively for small sizes.

def _sqr_chunk_terms(j0, Q):
    """(k, i, j, weight) terms the kernel forms for column chunk j0."""
    terms = []
    cm = j0 // 2
    for c in range(cm + 1):
        for s in range(Q):
            for q in range(Q):
                i = Q * c + s
                k = Q * j0 + q
                j = k - i
                if j < 0:
                    continue  # B's zero prefix
                if c < cm:
                    terms.append((k, i, j, 2))
                else:
                    key = 2 * s - q - (Q if j0 & 1 else 0)
                    if key < 0:
                        terms.append((k, i, j, 2))
                    elif key == 0:
                        terms.append((k, i, j, 1))
    return terms


@pytest.mark.parametrize("M,Q", [(16, 4), (32, 4), (64, 4), (32, 8), (64, 8)])
def test_square_block_selection(M, Q):
    rng = random.Random(M * Q)
    a = [rng.getrandbits(32) for _ in range(M)]
    for j0 in range(M // Q):
        got = {}
        for k, i, j, w in _sqr_chunk_terms(j0, Q):
            assert i < j or (i == j and w == 1), (j0, k, i, j, w)
            got[k] = got.get(k, 0) + w * a[i] * a[j]
        for q in range(Q):
            k = Q * j0 + q
            want = sum(a[i] * a[k - i] for i in range(k + 1))
            assert got.get(k, 0) == want, (M, Q, j0, k)


# ---------------------------------------------------------------------------
# pair_conv_shfl (mul_ntt.cu, 2^20-bit cluster NTT): the last forward DIF
# stage and the first inverse DIT stage have twiddle 1; with the pointwise
# Montgomery product between them they are replaced by c0 = S + D,
# c1 = S - D + 2p with S = mont(a0 + a1, b0 + b1), D = mont(a0 - a1, b0 - b1)
# (lazy-reduced).  The replacement must be bit-identical to the three steps
# it removes (fwd stage w = 1 on both vectors, mont, inv stage w = 1) for
# every input the forward pass can hand over, i.e. all values in [0, 2p).

def _stage_sequence(a0, a1, b0, b1, p):
    p2 = 2 * p
    fa0, fa1 = red2((a0 + a1) & MASK, p2), red2((a0 - a1 + p2) & MASK, p2)   # fwd_pass, w^0
    fb0, fb1 = red2((b0 + b1) & MASK, p2), red2((b0 - b1 + p2) & MASK, p2)
    c0, c1 = mont(fa0, fb0, p), mont(fa1, fb1, p)                            # pointwise
    u, v = red2(c0, p2), red2(c1, p2)                                        # inv_pass, w^0
    return (u + v) & MASK, (u - v + p2) & MASK


def _pair_conv(a0, a1, b0, b1, p):
    p2 = 2 * p
    S = mont(red2((a0 + a1) & MASK, p2), red2((b0 + b1) & MASK, p2), p)
    D = mont(red2((a0 - a1 + p2) & MASK, p2), red2((b0 - b1 + p2) & MASK, p2), p)
    return (S + D) & MASK, (S - D + p2) & MASK


def test_pair_conv_equals_stage_sequence():
    rng = random.Random(20)
    for p in PRIMES:
        p2 = 2 * p
        edge = [0, 1, p - 1, p, p + 1, p2 - 1]
        vals = [(x, y, z, w) for x in edge for y in edge for z in (0, p2 - 1) for w in (1, p)]
        vals += [tuple(rng.randrange(p2) for _ in range(4)) for _ in range(4000)]
        for a0, a1, b0, b1 in vals:
            got = _pair_conv(a0, a1, b0, b1, p)
            assert got == _stage_sequence(a0, a1, b0, b1, p)
            assert max(got) < 4 * p                     # the inverse pass's input bound
            # and it is the 2-point cyclic convolution, times 2 R^-1 (R = 2^32)
            rinv = pow(1 << 32, -1, p)
            assert got[0] % p == 2 * (a0 * b0 + a1 * b1) * rinv % p
            assert got[1] % p == 2 * (a0 * b1 + a1 * b0) * rinv % p
