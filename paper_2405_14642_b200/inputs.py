"""Seeded synthetic operand generator shared by tests, smoke() and bench.py.

Holds none of the method's arithmetic: it only draws limb patterns.  The
same torch code runs on CPU (for the oracle side) and on CUDA (to create
bench inputs directly in HBM), and produces identical bits on both, because
it is a pure function of (seed, operand, global instance, limb) —
a counter-based splitmix64 hash (Steele, Lea & Flood 2014), evaluated in
int64 two's-complement arithmetic.

Input classes (the paper does not state its inputs,
reading R21 in DESIGN.md):

* ``U``      uniform random limbs.
* ``ONES``   a = b = 2^B - 1 (maximal NTT coefficients, sum = [FF..FE, FF..]).
* ``RIPPLE`` a = 2^B - 1, b = 1: a carry chain through every thread, warp
             and CTA boundary (PAPER.md:136-142's "pathological case").
* ``RUNS``   a uniform, b_i = ~a_i except with probability 1/64 where
             b_i = ~a_i + 1: geometric carry chains crossing chunk boundaries.
* ``SPARSE`` one set bit per operand at a random position.
* ``MIX``    per instance, one of the classes above (chosen by hash).

Limbs are returned as ``torch.int32`` tensors of shape [n_inst, m] whose bit
patterns are the u32 limbs (little-endian).
"""
from __future__ import annotations

import numpy as np
import torch

CLASSES = ("U", "ONES", "RIPPLE", "RUNS", "SPARSE", "MIX")
_BASIC = ("U", "ONES", "RIPPLE", "RUNS", "SPARSE")

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    c &= _M64
    return c - (1 << 64) if c >= (1 << 63) else c


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 bit patterns (wrapping arithmetic)."""
    z = z + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _key(seed: int, operand: int) -> int:
    z = torch.tensor([_s64(seed * 8 + operand)], dtype=torch.int64)
    return int(splitmix64(z).item())


def _hash_grid(seed: int, operand: int, inst0: int, n_inst: int, m: int, device) -> torch.Tensor:
    """u32 hash (as int64 in [0, 2^32)) for every (instance, limb)."""
    inst = torch.arange(inst0, inst0 + n_inst, dtype=torch.int64, device=device).view(-1, 1)
    limb = torch.arange(m, dtype=torch.int64, device=device).view(1, -1)
    if m <= 8192:
        ctr = (inst << 14) | limb  # m <= 8192 < 2^14
    elif m <= 32768:  # cluster sizes: m < 2^16, separate counter domain (bit 62)
        ctr = (inst << 16) | limb | (1 << 62)
    else:  # bn_add_big sizes: m <= 2^25 < 2^26, another domain (bit 61)
        ctr = (inst << 26) | limb | (1 << 61)
    return _lsr(splitmix64(ctr ^ _key(seed, operand)), 32)


def _to_i32(x: torch.Tensor) -> torch.Tensor:
    x = x & 0xFFFFFFFF
    return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32)


def _per_inst_hash(seed: int, salt: int, inst0: int, n_inst: int, device) -> torch.Tensor:
    inst = torch.arange(inst0, inst0 + n_inst, dtype=torch.int64, device=device)
    return _lsr(splitmix64(inst ^ _key(seed, salt)), 32)


def _class_limbs(cls: str, seed: int, inst0: int, n: int, m: int, device):
    full = torch.full((n, m), 0xFFFFFFFF, dtype=torch.int64, device=device)
    if cls == "U":
        return _hash_grid(seed, 0, inst0, n, m, device), _hash_grid(seed, 1, inst0, n, m, device)
    if cls == "ONES":
        return full, full.clone()
    if cls == "RIPPLE":
        b = torch.zeros((n, m), dtype=torch.int64, device=device)
        b[:, 0] = 1
        return full, b
    if cls == "RUNS":
        a = _hash_grid(seed, 0, inst0, n, m, device)
        bump = (_hash_grid(seed, 2, inst0, n, m, device) & 63) == 0
        b = ((a ^ 0xFFFFFFFF) + bump.to(torch.int64)) & 0xFFFFFFFF
        return a, b
    if cls == "SPARSE":
        out = []
        for op in (0, 1):
            pos = _per_inst_hash(seed, 16 + op, inst0, n, device) % (32 * m)
            x = torch.zeros((n, m), dtype=torch.int64, device=device)
            x.scatter_(1, (pos // 32).view(-1, 1), (1 << (pos % 32)).view(-1, 1))
            out.append(x)
        return out[0], out[1]
    raise ValueError("unknown input class %r (one of %s)" % (cls, CLASSES))


def make_operands(n_inst: int, m: int, seed: int = 1, cls: str = "U", inst0: int = 0,
                  device="cpu"):
    """Return (a, b) int32 tensors [n_inst, m] for global instances
    [inst0, inst0 + n_inst).  Bit-identical on every device and for every
    sharding of the instance range."""
    if cls not in CLASSES:
        raise ValueError("unknown input class %r (one of %s)" % (cls, CLASSES))
    if m < 1 or m > (1 << 25):
        raise ValueError("m must be in [1, 2^25]")
    if n_inst == 0:
        z = torch.zeros((0, m), dtype=torch.int32, device=device)
        return z, z.clone()
    if cls != "MIX":
        a, b = _class_limbs(cls, seed, inst0, n_inst, m, device)
        return _to_i32(a), _to_i32(b)
    pick = _per_inst_hash(seed, 31, inst0, n_inst, device) % len(_BASIC)
    a = torch.empty((n_inst, m), dtype=torch.int64, device=device)
    b = torch.empty_like(a)
    for ci, c in enumerate(_BASIC):
        ca, cb = _class_limbs(c, seed, inst0, n_inst, m, device)
        sel = (pick == ci).view(-1, 1)
        a = torch.where(sel, ca, a)
        b = torch.where(sel, cb, b)
    return _to_i32(a), _to_i32(b)


def to_numpy_u32(x: torch.Tensor) -> np.ndarray:
    """int32 bit patterns -> contiguous uint32 numpy array (host)."""
    return x.detach().cpu().contiguous().numpy().view(np.uint32)


def from_numpy_u32(x: np.ndarray, device="cpu") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).to(device)
