"""Paper §4 (FFT multiplication) written out step by step — TEST INFRASTRUCTURE ONLY.

Only tests/ (and smoke/bench cpu legs) may import this; the product path
never does, and this module imports nothing from it.

Pure-Python integers, small sizes only.  Each function cites the passage it
follows; where the paper is garbled or inexact the DESIGN.md reading is named.

* ``is_prime``                — deterministic Miller–Rabin (64-bit), textbook.
* ``first_root_of_order``     — §4.1: "iterate through the
  elements a of Z_p and chose the first one (if any) that also verifies
  g^q != 1 for all q < 2^n".  Reading R15: g is the first a >= 2
  whose multiplicative order is exactly 2^n (reproduces g = 13 and g = 21 of
  PAPER.md:710-711; the "g = a^k" reading of PAPER.md:668 does not).
* ``omega``                   — PAPER.md:670-674: omega = g^(2^n / M).
* ``omegas_table``            — PAPER.md:807-809: exclusive scan of P::mul
  over replicate M omega, i.e. [1, w, w^2, ...].
* ``zmod_add/sub/mul``        — Fig. 8, PAPER.md:686-699 (norm/mul read as
  r % modulus, reading R12).
* ``dft_direct``              — the definition X_k = sum_i x_i w^(ik) mod p.
* ``fft_fig9`` / ``ifft_fig9`` — Fig. 9: bit-reverse
  permutation then lg M radix-2 DIT stages with twiddle omegas[r*j],
  r = M >> t; ifft = fft with omegas_inv then scale by invM.
* ``max_exact_digit_width``   — the exactness bound n*(2^d-1)^2 < p that the
  paper's digit scheme must satisfy (reading R10).
* ``fft_mul_paper``           — bmulFFT as printed: an
  M-point *cyclic* transform over d-bit digits, no zero padding (reading
  R11) — used only as the negative control showing the printed scheme is
  inexact at the paper's sizes.
* ``fft_mul_padded`` / ``fft_mul_exact`` — the exact reading the build implements
  (R10/R11): zero-pad to N = 2m, one transform per prime, CRT — written
  with direct DFTs for tiny m so it checks the reading, not the kernels.
"""
from __future__ import annotations

from typing import List, Sequence

# PAPER.md:709-712, the two "good" primes found by the authors' Maple search.
PRIME_FIELD_32 = dict(p=3221225473, k=3, n=30, g=13)
PRIME_FIELD_64 = dict(p=4179340454199820289, k=29, n=57, g=21)


def is_prime(n: int) -> bool:
    """Deterministic Miller–Rabin for n < 3.3e24 (bases = first 13 primes)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for q in small:
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def order_is_exactly(a: int, p: int, n: int) -> bool:
    """a^(2^n) == 1 and a^(2^(n-1)) != 1  (order exactly 2^n)."""
    return pow(a, 1 << n, p) == 1 and pow(a, 1 << (n - 1), p) != 1


def first_root_of_order(p: int, n: int, limit: int = 1 << 20) -> int:
    """§4.1, reading R15: first a >= 2 of order exactly 2^n."""
    for a in range(2, min(p, limit)):
        if order_is_exactly(a, p, n):
            return a
    raise ValueError("no element of order 2^%d below %d" % (n, limit))


def omega(p: int, g: int, n: int, M: int) -> int:
    """omega = g^(2^n / M) for a power-of-two M <= 2^n."""
    assert M & (M - 1) == 0 and M <= (1 << n)
    return pow(g, (1 << n) // M, p)


def omegas_table(p: int, w: int, M: int) -> List[int]:
    """scan^exc (P::mul) 1 (replicate M w)."""
    out, acc = [], 1
    for _ in range(M):
        out.append(acc)
        acc = acc * w % p
    return out


# Fig. 8
def zmod_add(x: int, y: int, p: int) -> int:
    r = x + y
    if r >= p:
        r -= p
    return r


def zmod_sub(x: int, y: int, p: int) -> int:
    r = x
    if x < y:
        r += p
    return r - y


def zmod_mul(x: int, y: int, p: int) -> int:
    return (x * y) % p


def dft_direct(x: Sequence[int], w: int, p: int) -> List[int]:
    """X_k = sum_i x_i w^(i k) mod p — the definition, O(N^2)."""
    N = len(x)
    return [sum(x[i] * pow(w, i * k, p) for i in range(N)) % p for k in range(N)]


def _bitrev(i: int, lg: int) -> int:
    r = 0
    for _ in range(lg):
        r = (r << 1) | (i & 1)
        i >>= 1
    return r


def fft_fig9(x: Sequence[int], omegas: Sequence[int], p: int) -> List[int]:
    """Fig. 9 ``fft``: permute, then for t = 1..lgM:
    L = 2^t, Ld2 = L/2, r = M >> t; each butterfly k*L + j (j < Ld2) uses
    omega_pow = omegas[r*j], tau = omega_pow * x[kLj + Ld2],
    x[kLj] = x[kLj] + tau, x[kLj + Ld2] = x[kLj] - tau."""
    M = len(x)
    lgM = M.bit_length() - 1
    assert 1 << lgM == M
    sh = [x[_bitrev(i, lgM)] for i in range(M)]  # permute
    for t in range(1, lgM + 1):
        L, Ld2, r = 1 << t, 1 << (t - 1), M >> t
        for vtid in range(M // 2):
            k = vtid >> (t - 1)
            j = vtid & (Ld2 - 1)
            kLj = k * L + j
            tau = zmod_mul(omegas[r * j], sh[kLj + Ld2], p)
            xk = sh[kLj]
            sh[kLj] = zmod_add(xk, tau, p)
            sh[kLj + Ld2] = zmod_sub(xk, tau, p)
    return sh


def ifft_fig9(x: Sequence[int], omegas_inv: Sequence[int], invM: int, p: int) -> List[int]:
    """Fig. 9 ``ifft``: fft with omegas_inv, then * invM."""
    return [zmod_mul(invM, v, p) for v in fft_fig9(x, omegas_inv, p)]


def max_exact_digit_width(p: int, n_terms: int, max_d: int = 64) -> int:
    """Largest d with n_terms * (2^d - 1)^2 < p: the widest digit for which a
    length-n cyclic convolution coefficient cannot wrap mod p (reading R10)."""
    best = 0
    for d in range(1, max_d + 1):
        if n_terms * ((1 << d) - 1) ** 2 < p:
            best = d
    return best


def _digits(v: int, d: int, count: int) -> List[int]:
    mask = (1 << d) - 1
    return [(v >> (d * i)) & mask for i in range(count)]


def fft_mul_paper(A: int, B: int, n_digits: int, d: int, field: dict) -> int:
    """bmulFFT as printed: split A, B into n_digits
    d-bit digits, M = n_digits point *cyclic* transform (no zero padding),
    pointwise product, inverse, then carry the coefficients in base 2^d.
    Returns the value mod 2^(d * n_digits).  Negative control only."""
    p, n, g = field["p"], field["n"], field["g"]
    M = n_digits
    w = omega(p, g, n, M)
    winv = pow(w, p - 2, p)
    om, omi = omegas_table(p, w, M), omegas_table(p, winv, M)
    fa = fft_fig9(_digits(A, d, M), om, p)
    fb = fft_fig9(_digits(B, d, M), om, p)
    t = [zmod_mul(u, v, p) for u, v in zip(fa, fb)]
    c = ifft_fig9(t, omi, pow(M, p - 2, p), p)
    return sum(ci << (d * i) for i, ci in enumerate(c)) % (1 << (d * M))


def fft_mul_padded(A: int, B: int, n_digits: int, d: int, primes: Sequence[int]) -> int:
    """Zero-padded (acyclic) NTT product on d-bit digits, truncated to
    n_digits digits, with direct DFTs (tiny sizes only): pad both digit
    vectors to N = the power of two >= 2 n_digits, per prime p:
    c_p = DFT^-1(DFT(a) * DFT(b)); CRT the residues to one coefficient per
    position (plain sum r * Mp * (Mp^-1 mod p) mod P); carry in base 2^d.
    Exact iff prod(primes) > n_digits * (2^d - 1)^2 (reading R10)."""
    N = 1
    while N < 2 * n_digits:
        N *= 2
    a = _digits(A, d, n_digits) + [0] * (N - n_digits)
    b = _digits(B, d, n_digits) + [0] * (N - n_digits)
    P = 1
    for p in primes:
        P *= p
    coeff = [0] * N
    for p in primes:
        assert (p - 1) % N == 0, "prime %d has no %d-th root of unity" % (p, N)
        # an element of order exactly N: g^((p-1)/N) for a primitive root g
        g = next(x for x in range(2, 1000)
                 if all(pow(x, (p - 1) // q, p) != 1 for q in _prime_factors(p - 1)))
        w = pow(g, (p - 1) // N, p)
        fa, fb = dft_direct(a, w, p), dft_direct(b, w, p)
        t = [u * v % p for u, v in zip(fa, fb)]
        c = dft_direct(t, pow(w, p - 2, p), p)
        ninv = pow(N, p - 2, p)
        Mp = P // p
        for k in range(N):
            coeff[k] += (c[k] * ninv % p) * Mp * pow(Mp, p - 2, p)
    coeff = [v % P for v in coeff]
    return sum(ck << (d * k) for k, ck in enumerate(coeff)) % (1 << (d * n_digits))


def fft_mul_exact(A: int, B: int, m: int, primes: Sequence[int]) -> int:
    """The exact reading (R10/R11) on 32-bit limbs: fft_mul_padded with
    d = 32 and enough primes that prod(primes) > m * (2^32 - 1)^2."""
    P = 1
    for p in primes:
        P *= p
    assert P > m * ((1 << 32) - 1) ** 2, "CRT range too small for exact coefficients"
    return fft_mul_padded(A, B, m, 32, primes)


def _prime_factors(n: int) -> List[int]:
    out, q = [], 2
    while q * q <= n:
        if n % q == 0:
            out.append(q)
            while n % q == 0:
                n //= q
        q += 1
    if n > 1:
        out.append(n)
    return out
