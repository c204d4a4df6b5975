"""Pins for oracle/ntt_ref.py (paper §4 written out) — run with -m "not gpu".

Pinned against: the paper's printed constants (tests/golden/paper_constants.txt),
the DFT definition and its closed forms (delta -> ones, ones -> N*delta),
brute-force cyclic convolution, Python-int products, and SPEC's derived
exactness bounds.
"""
import os
import random

import pytest

from oracle import ntt_ref as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _constants():
    rows = []
    with open(os.path.join(GOLDEN, "paper_constants.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                name, p, k, n, g = line.split()
                rows.append((name, int(p), int(k), int(n), int(g)))
    return rows


@pytest.mark.parametrize("row", _constants(), ids=lambda r: r[0])
def test_paper_prime_fields(row):
    name, p, k, n, g = row
    assert p == k * (1 << n) + 1                  # PAPER.md:660 shape
    assert R.is_prime(p)
    assert R.order_is_exactly(g, p, n)            # g^(2^n) = 1, g^(2^(n-1)) != 1
    assert R.first_root_of_order(p, n) == g       # reading R15 reproduces the printed g
    assert (R.PRIME_FIELD_32 if name.endswith("32") else R.PRIME_FIELD_64)["g"] == g


def test_gak_reading_does_not_reproduce_g():
    """The literal 'g = a^k' reading of PAPER.md:668 (first a whose a^k has order 2^n)
    gives a different g — the reason DESIGN.md takes reading R15."""
    f = R.PRIME_FIELD_32
    a = next(a for a in range(2, 100) if R.order_is_exactly(pow(a, f["k"], f["p"]), f["p"], f["n"]))
    assert pow(a, f["k"], f["p"]) != f["g"]


def test_is_prime_small_table():
    primes = [x for x in range(2, 400) if all(x % d for d in range(2, int(x ** 0.5) + 1))]
    assert [x for x in range(400) if R.is_prime(x)] == primes


def test_omega_is_primitive():
    f = R.PRIME_FIELD_32
    for M in (2, 8, 64, 1 << 12):
        w = R.omega(f["p"], f["g"], f["n"], M)
        assert pow(w, M, f["p"]) == 1 and pow(w, M // 2, f["p"]) == f["p"] - 1


SMALL_FIELDS = [(257, 3), (7681, 17), (12289, 11), (R.PRIME_FIELD_32["p"], R.PRIME_FIELD_32["g"])]


def _root(p, N):
    # an element of order exactly N (p-1 divisible by N)
    for a in range(2, p):
        w = pow(a, (p - 1) // N, p)
        if pow(w, N // 2, p) == p - 1:
            return w
    raise AssertionError


@pytest.mark.parametrize("p,_g", SMALL_FIELDS)
def test_dft_closed_forms(p, _g):
    for N in (2, 4, 16, 64):
        w = _root(p, N)
        delta = [1] + [0] * (N - 1)
        assert R.dft_direct(delta, w, p) == [1] * N
        assert R.dft_direct([1] * N, w, p) == [N % p] + [0] * (N - 1)


@pytest.mark.parametrize("p,_g", SMALL_FIELDS)
def test_fig9_fft_equals_dft(p, _g):
    rng = random.Random(p)
    for N in (2, 4, 8, 32, 64):
        w = _root(p, N)
        x = [rng.randrange(p) for _ in range(N)]
        assert R.fft_fig9(x, R.omegas_table(p, w, N), p) == R.dft_direct(x, w, p)


@pytest.mark.parametrize("p,_g", SMALL_FIELDS)
def test_roundtrip_and_convolution_theorem(p, _g):
    rng = random.Random(p + 1)
    for N in (4, 16, 64, 256):
        if (p - 1) % N:
            continue
        w = _root(p, N)
        wi = pow(w, p - 2, p)
        om, omi, invN = R.omegas_table(p, w, N), R.omegas_table(p, wi, N), pow(N, p - 2, p)
        x = [rng.randrange(p) for _ in range(N)]
        y = [rng.randrange(p) for _ in range(N)]
        assert R.ifft_fig9(R.fft_fig9(x, om, p), omi, invN, p) == x
        cyc = [sum(x[i] * y[(k - i) % N] for i in range(N)) % p for k in range(N)]
        fx, fy = R.fft_fig9(x, om, p), R.fft_fig9(y, om, p)
        assert R.ifft_fig9([u * v % p for u, v in zip(fx, fy)], omi, invN, p) == cyc


def test_exact_digit_width_bounds():
    """SPEC.md:428-430 derived values (exact integer checks)."""
    assert R.max_exact_digit_width(R.PRIME_FIELD_32["p"], 3) == 15
    assert R.max_exact_digit_width(R.PRIME_FIELD_32["p"], 4) == 14
    assert R.max_exact_digit_width(R.PRIME_FIELD_64["p"], 1 << 17) == 22
    # reading R10: the paper's widths (15 with PF32, 31 with PF64) are not exact
    # at any of its sizes (>= 2^11 bits -> >= 137 15-bit digits):
    assert R.max_exact_digit_width(R.PRIME_FIELD_32["p"], 137) < 15
    assert (2**31 - 1) ** 2 > R.PRIME_FIELD_64["p"]


def test_paper_scheme_negative_control():
    """SPEC acceptance 6: PF32, conv length 4, all-max 15-bit digits -> wrong;
    14-bit digits -> right (the bound is sharp, the paper's width is inexact)."""
    p = R.PRIME_FIELD_32["p"]
    n = 4
    for d, ok in ((15, False), (14, True)):
        A = (1 << (d * n)) - 1        # all-max digits: coefficient 3 has 4 max terms
        got = R.fft_mul_padded(A, A, n, d, [p])
        assert (got == (A * A) % (1 << (d * n))) is ok
    # and with 3 digits the 15-bit width is still exact
    A = (1 << 45) - 1
    assert R.fft_mul_padded(A, A, 3, 15, [p]) == (A * A) % (1 << 45)


def test_cyclic_no_padding_is_wrong():
    """Reading R11: an M-point cyclic transform on M digits wraps the high
    coefficients onto the low ones even when digits are small."""
    f = R.PRIME_FIELD_32
    d, n = 8, 8
    A = (1 << (d * n)) - 1
    assert R.fft_mul_paper(A, A, n, d, f) != (A * A) % (1 << (d * n))


def _cyclic_product_by_hand(A, B, M, d, p):
    """The value bmulFFT must return, written without any
    transform: digits a_i, b_j of A, B (d bits, M of them); the cyclic
    coefficient c_k = sum over i + j == k (mod M) of a_i * b_j, reduced mod p;
    then sum c_k 2^(d k) carried mod 2^(d M) (M-point transform
    on M digits, no zero padding)."""
    a = [(A >> (d * i)) & ((1 << d) - 1) for i in range(M)]
    b = [(B >> (d * j)) & ((1 << d) - 1) for j in range(M)]
    c = [0] * M
    for i in range(M):
        for j in range(M):
            c[(i + j) % M] += a[i] * b[j]
    return sum((ck % p) << (d * k) for k, ck in enumerate(c)) % (1 << (d * M))


@pytest.mark.parametrize("field", ["PF32", "PF64"])
@pytest.mark.parametrize("M", [4, 8, 16])
def test_fft_mul_paper_is_cyclic_convolution(field, M):
    """Pin of fft_mul_paper (bmulFFT as printed):
    it must equal the cyclic convolution of the digit vectors mod p, carried
    in base 2^d — computed by the double loop above, no DFT involved.  A
    wrong inverse twiddle direction (c_k -> c_{-k}), a missing or wrong invM,
    or a dropped wrap term all change the result on these random digits."""
    f = R.PRIME_FIELD_32 if field == "PF32" else R.PRIME_FIELD_64
    p = f["p"]
    rng = random.Random(1000 * M + (32 if field == "PF32" else 64))
    for d in (8, 15) if field == "PF32" else (16, 31):
        for _ in range(4):
            A, B = rng.getrandbits(d * M), rng.getrandbits(d * M)
            assert R.fft_mul_paper(A, B, M, d, f) == _cyclic_product_by_hand(A, B, M, d, p)
        # coefficients that exceed p (all-max digits) are reduced mod p, not kept
        A = (1 << (d * M)) - 1
        assert R.fft_mul_paper(A, A, M, d, f) == _cyclic_product_by_hand(A, A, M, d, p)


@pytest.mark.parametrize("field", ["PF32", "PF64"])
def test_fft_mul_paper_exact_when_wrap_vanishes(field):
    """Positive case of bmulFFT: when A has a single nonzero digit (A < 2^d),
    c_k = a_0 b_k, nothing wraps and nothing exceeds p, so the printed
    scheme returns the true product A*B mod 2^(dM) (Eq. 1)."""
    f = R.PRIME_FIELD_32 if field == "PF32" else R.PRIME_FIELD_64
    rng = random.Random(7)
    d = 12 if field == "PF32" else 24
    for M in (4, 8, 16):
        for _ in range(3):
            A, B = rng.getrandbits(d), rng.getrandbits(d * M)
            assert R.fft_mul_paper(A, B, M, d, f) == (A * B) % (1 << (d * M))
        assert R.fft_mul_paper(1, B, M, d, f) == B


def _find_primes(count, lo_bits=29, hi=1 << 30, two_adicity=15):
    out, k = [], (hi - 1) >> two_adicity
    while len(out) < count:
        p = k * (1 << two_adicity) + 1
        if p < hi and p.bit_length() > lo_bits and R.is_prime(p):
            out.append(p)
        k -= 1
    return out


@pytest.mark.parametrize("m", [1, 2, 3, 4, 8])
def test_exact_reading_three_primes(m):
    """Readings R10/R11: zero padding to 2m and 3 primes < 2^30 + CRT give the
    exact truncated product on 32-bit digits, including all-ones inputs."""
    primes = _find_primes(3)
    rng = random.Random(m)
    mod = 1 << (32 * m)
    cases = [(mod - 1, mod - 1), (mod - 1, 1)] + [(rng.randrange(mod), rng.randrange(mod)) for _ in range(3)]
    for A, B in cases:
        assert R.fft_mul_exact(A, B, m, primes) == (A * B) % mod


def test_metric_formulas_golden():
    """PAPER.md:929 and :935 (tests/golden/metric_formulas.txt)."""
    with open(os.path.join(GOLDEN, "metric_formulas.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                bits, insts, nbytes, ops = map(int, line.split())
                m = bits // 32
                assert 3 * insts * bits // 8 == nbytes
                assert 300 * m * (m.bit_length() - 1) == ops
                assert bits * insts == 2**32
