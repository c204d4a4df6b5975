"""Pins for the CPU oracle (oracle/oracle.c) — run with -m "not gpu".

The oracle is pinned to things other than itself:
* Python's arbitrary-precision int (an independent big-int runtime),
* exhaustive brute force over a 16-value limb alphabet for m = 1, 2,
* closed forms and algebraic invariants,
* the worked examples in tests/golden/worked_examples.txt (cited there).
"""
import os
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_14642_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

ALPHABET = [0, 1, 2, 3, 0x0000FFFF, 0xFFFF0000, 0x55555555, 0xAAAAAAAA, 0x12345678,
            0xDEADBEEF, 0x7FFFFFFF, 0x80000000, 0x80000001, 0xFFFFFFFD, 0xFFFFFFFE,
            0xFFFFFFFF]


def to_int(limbs) -> int:
    v = 0
    for i, x in enumerate(np.asarray(limbs, dtype=np.uint64).tolist()):
        v |= int(x) << (32 * i)
    return v


def from_int(v: int, m: int) -> np.ndarray:
    return np.array([(v >> (32 * i)) & 0xFFFFFFFF for i in range(m)], dtype=np.uint32)


def rows_to_ints(x: np.ndarray):
    return [to_int(r) for r in x]


# ---------------------------------------------------------------- golden

def _golden_rows():
    rows = []
    with open(os.path.join(GOLDEN, "worked_examples.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            op, a, b, out = [s.strip() for s in line.split("|")]
            parse = lambda s: np.array([int(t, 16) for t in s.split()], dtype=np.uint32)
            rows.append((op, parse(a), parse(b), parse(out)))
    return rows


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: r[0] + str(len(r[1])))
def test_worked_examples(row):
    op, a, b, out = row
    got = (O.add if op == "add" else O.mul)(a, b)[0]
    assert np.array_equal(got, out)


# ------------------------------------------------------ exhaustive / closed form

@pytest.mark.parametrize("m", [1, 2])
def test_exhaustive_alphabet(m):
    """Every pair of m-limb numbers over the 16-value limb alphabet:
    m=1 -> 256 pairs, m=2 -> 65,536 pairs, against Python ints."""
    vals = np.array(ALPHABET, dtype=np.uint32)
    if m == 1:
        xs = vals.reshape(-1, 1)
    else:
        xs = np.stack(np.meshgrid(vals, vals, indexing="ij"), -1).reshape(-1, 2)
    n = xs.shape[0]
    a = np.repeat(xs, n, axis=0)
    b = np.tile(xs, (n, 1))
    s, p = O.add(a, b), O.mul(a, b)
    mod = 1 << (32 * m)
    ai, bi = rows_to_ints(a), rows_to_ints(b)
    assert rows_to_ints(s) == [(x + y) % mod for x, y in zip(ai, bi)]
    assert rows_to_ints(p) == [(x * y) % mod for x, y in zip(ai, bi)]


def test_random_three_limb():
    rng = np.random.default_rng(7)
    a = rng.integers(0, 2**32, size=(200000, 3), dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, size=(200000, 3), dtype=np.uint64).astype(np.uint32)
    # bias some limbs to the extremes so carries ripple
    a[::3, 1] = 0xFFFFFFFF
    b[::5, 0] = 0xFFFFFFFF
    s, p = O.add(a, b, nthreads=4), O.mul(a, b, nthreads=4)
    mod = 1 << 96
    ai, bi = rows_to_ints(a), rows_to_ints(b)
    assert rows_to_ints(s) == [(x + y) % mod for x, y in zip(ai, bi)]
    assert rows_to_ints(p) == [(x * y) % mod for x, y in zip(ai, bi)]


@pytest.mark.parametrize("m", [32, 128, 1024, 8192])
@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "RUNS", "SPARSE"])
def test_python_int(m, cls):
    n = 4 if m <= 1024 else 1
    a, b = inputs.make_operands(n, m, seed=11, cls=cls)
    a, b = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    mod = 1 << (32 * m)
    ai, bi = rows_to_ints(a), rows_to_ints(b)
    assert rows_to_ints(O.add(a, b)) == [(x + y) % mod for x, y in zip(ai, bi)]
    assert rows_to_ints(O.mul(a, b)) == [(x * y) % mod for x, y in zip(ai, bi)]


# ------------------------------------------------------------- invariants

def _rand(m, n=8, seed=3):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 2**32, size=(n, m), dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("m", [1, 5, 64, 333])
def test_add_invariants(m):
    a, b = _rand(m, seed=1), _rand(m, seed=2)
    ones = np.full_like(a, 0xFFFFFFFF)
    one = np.zeros_like(a)
    one[:, 0] = 1
    assert np.array_equal(O.add(a, b), O.add(b, a))                       # commutative
    nb = ~b
    assert np.array_equal(O.add(O.add(O.add(a, b), nb), one), a)          # (a+b)-b = a
    assert np.array_equal(O.add(a, ~a), ones)                             # a + ~a = 2^B-1
    for r in range(a.shape[0]):
        s, c = O.add_carry(O.add(a[r], ~a[r])[0], one[r])
        assert not s.any() and c == 1                                     # a + ~a + 1 = 2^B
    assert not O.add(ones, one).any()                                     # all-ones + 1 = 0
    assert np.array_equal(O.add(a, np.zeros_like(a)), a)


@pytest.mark.parametrize("m", [1, 4, 64, 257])
def test_mul_invariants(m):
    a, b, c = _rand(m, seed=4), _rand(m, seed=5), _rand(m, seed=6)
    one = np.zeros_like(a)
    one[:, 0] = 1
    ones = np.full_like(a, 0xFFFFFFFF)
    assert np.array_equal(O.mul(a, b), O.mul(b, a))
    assert np.array_equal(O.mul(a, one), a)
    assert not O.mul(a, np.zeros_like(a)).any()
    assert np.array_equal(O.mul(a, O.add(b, c)), O.add(O.mul(a, b), O.mul(a, c)))
    assert np.array_equal(O.mul(ones, ones), one)                         # (2^B-1)^2 = 1 mod 2^B


def test_powers_of_two():
    m = 16
    for i in range(0, 32 * m, 37):
        for j in range(0, 32 * m, 41):
            a, b = from_int(1 << i, m), from_int(1 << j, m)
            want = from_int((1 << (i + j)) % (1 << (32 * m)), m)
            assert np.array_equal(O.mul(a, b)[0], want)


@pytest.mark.parametrize("q", [65521, 2**31 - 1, 10**9 + 7])
def test_full_product_residues(q):
    """full product mod q == (A mod q)(B mod q) mod q (Horner over limbs)."""
    def res(limbs):
        r = 0
        for x in reversed(np.asarray(limbs, dtype=np.uint64).tolist()):
            r = (r * (1 << 32) + int(x)) % q
        return r
    for m in (3, 50, 512):
        a, b = _rand(m, n=2, seed=m)[0], _rand(m, n=2, seed=m + 1)[1]
        full = O.mul_full(a, b)
        assert res(full) == res(a) * res(b) % q
        assert np.array_equal(full[:m], O.mul(a, b)[0])                   # truncation = low half


def test_batch_threads_agree():
    a, b = _rand(40, n=101, seed=9), _rand(40, n=101, seed=10)
    assert np.array_equal(O.mul(a, b, nthreads=1), O.mul(a, b, nthreads=7))
    assert np.array_equal(O.add(a, b, nthreads=1), O.add(a, b, nthreads=3))


def test_in_place_batch_and_empty():
    a = _rand(8, n=0)
    assert O.add(a, a).shape == (0, 8)
    with pytest.raises(ValueError):
        O.add(_rand(4), _rand(5))


# ------------------------------------------- fused workloads

@pytest.mark.parametrize("m", [1, 3, 32, 1024])
@pytest.mark.parametrize("cls", ["U", "ONES", "RIPPLE", "RUNS", "SPARSE"])
def test_fused_python_int(m, cls):
    """6-Add = 4A + 3B and Poly = (A A + B)(B B + B) + A B, both mod 2^(32m),
    against Python's arbitrary-precision ints (R17/R18)."""
    n = 5 if m <= 32 else 2
    a, b = inputs.make_operands(n, m, seed=m + len(cls), cls=cls)
    a, b = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    mod = 1 << (32 * m)
    ai, bi = rows_to_ints(a), rows_to_ints(b)
    assert rows_to_ints(O.add6(a, b)) == [(4 * x + 3 * y) % mod for x, y in zip(ai, bi)]
    assert rows_to_ints(O.poly(a, b, nthreads=2)) == \
        [((x * x + y) * (y * y + y) + x * y) % mod for x, y in zip(ai, bi)]


def test_fused_exhaustive_alphabet_one_limb():
    """m = 1: all 256 alphabet pairs against u64 arithmetic mod 2^32."""
    pairs = [(x, y) for x in ALPHABET for y in ALPHABET]
    a = np.array([[x] for x, _ in pairs], dtype=np.uint32)
    b = np.array([[y] for _, y in pairs], dtype=np.uint32)
    M = 1 << 32
    want6 = [(4 * x + 3 * y) % M for x, y in pairs]
    wantp = [((x * x + y) % M * ((y * y + y) % M) + x * y) % M for x, y in pairs]
    assert O.add6(a, b)[:, 0].tolist() == want6
    assert O.poly(a, b)[:, 0].tolist() == wantp


@pytest.mark.parametrize("m", [4, 128])
def test_fused_closed_forms(m):
    """Special cases with closed forms: a = b = 2^B - 1 = -1 (mod 2^B):
    6-Add = -7, Poly = (1 - 1)(1 - 1) + 1 = 1; b = 0: 6-Add = 4a, Poly = 0;
    a = 0: Poly = b^3 + b^2; b = 1: Poly = 2a^2 + a + 2."""
    rng = np.random.default_rng(m)
    a = rng.integers(0, 2**32, size=(3, m), dtype=np.uint64).astype(np.uint32)
    ones = np.full_like(a, 0xFFFFFFFF)
    zero = np.zeros_like(a)
    one = zero.copy()
    one[:, 0] = 1
    mod = 1 << (32 * m)
    assert rows_to_ints(O.add6(ones, ones)) == [mod - 7] * 3
    assert np.array_equal(O.poly(ones, ones), one)
    assert rows_to_ints(O.add6(a, zero)) == [4 * x % mod for x in rows_to_ints(a)]
    assert not O.poly(a, zero).any()
    assert rows_to_ints(O.poly(zero, a)) == [(y ** 3 + y ** 2) % mod for y in rows_to_ints(a)]
    assert rows_to_ints(O.poly(a, one)) == [(2 * x * x + x + 2) % mod for x in rows_to_ints(a)]


@pytest.mark.parametrize("m", [1, 2, 32, 1024])
@pytest.mark.parametrize("cls", ["U", "ONES", "RUNS", "SPARSE"])
def test_mul_full_python_int(m, cls):
    """Full 2m-limb product (the wide entry points' definition) against
    Python ints: A * B exactly, no truncation (Eq. 1 with k < 2M)."""
    n = 3 if m <= 32 else 1
    a, b = inputs.make_operands(n, m, seed=m + 5, cls=cls)
    a, b = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    got = O.mul_full_rows(a, b)
    assert got.shape == (n, 2 * m)
    assert rows_to_ints(got) == [x * y for x, y in zip(rows_to_ints(a), rows_to_ints(b))]
