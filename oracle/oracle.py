"""ctypes front-end to oracle.c — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2405_14642_b200``) never imports it, and it never imports the
product package: the two share no code (the seeded input generator lives in
its own module, ``paper_2405_14642_b200/inputs.py``, and holds none of the
method's arithmetic).

Functions (all over instance-major ``[n_inst, m]`` uint32 numpy arrays,
little-endian limbs):

* ``add(a, b)``       -> (A + B) mod 2^(32m)   (Fig. 1 left)
* ``mul(a, b)``       -> (A * B) mod 2^(32m)   (Eq. 1)
* ``mul_full(a, b)``  -> A * B as 2m limbs (for residue pins)
* ``add6(a, b)``      -> 6-Add, 4A + 3B mod 2^(32m) as six additions (R17)
* ``poly(a, b)``      -> Poly, ((A A + B)(B B + B) + A B) mod 2^(32m)
* ``add_carry(a, b)`` -> (sum, carry-out) of one instance (carry for tests)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ORACLE_ADD = 0
ORACLE_MUL = 1
ORACLE_ADD6 = 2
ORACLE_POLY = 3


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc into oracle/liboracle.so (plain -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u32p = ctypes.POINTER(ctypes.c_uint32)
            lib.oracle_add.argtypes = [u32p, u32p, u32p, ctypes.c_uint32]
            lib.oracle_add.restype = ctypes.c_uint32
            lib.oracle_mul.argtypes = [u32p, u32p, u32p, ctypes.c_uint32]
            lib.oracle_mul.restype = None
            lib.oracle_mul_full.argtypes = [u32p, u32p, u32p, ctypes.c_uint32]
            lib.oracle_mul_full.restype = None
            lib.oracle_batch.argtypes = [ctypes.c_int, u32p, u32p, u32p, ctypes.c_uint64,
                                         ctypes.c_uint32, ctypes.c_int]
            lib.oracle_batch.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(x: np.ndarray):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _as2d(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint32)
    return x.reshape(1, -1) if x.ndim == 1 else x


def _batch(op: int, a, b, nthreads: int) -> np.ndarray:
    a, b = _as2d(a), _as2d(b)
    if a.shape != b.shape:
        raise ValueError("operand shapes differ: %s vs %s" % (a.shape, b.shape))
    out = np.empty_like(a)
    n, m = a.shape
    if n and m:
        rc = _load().oracle_batch(op, _p(out), _p(a), _p(b), n, m, int(nthreads))
        if rc:
            raise RuntimeError("oracle_batch failed")
    return out


def add(a, b, nthreads: int = 1) -> np.ndarray:
    """(A + B) mod 2^(32m) per instance (rows)."""
    return _batch(ORACLE_ADD, a, b, nthreads)


def mul(a, b, nthreads: int = 1) -> np.ndarray:
    """(A * B) mod 2^(32m) per instance (rows)."""
    return _batch(ORACLE_MUL, a, b, nthreads)


def add6(a, b, nthreads: int = 1) -> np.ndarray:
    """6-Add: r = a + b, then + a, + b, + a, + b, + a, per instance (rows)."""
    return _batch(ORACLE_ADD6, a, b, nthreads)


def poly(a, b, nthreads: int = 1) -> np.ndarray:
    """Poly: ((a a + b)(b b + b) + a b) mod 2^(32m) per instance (rows)."""
    return _batch(ORACLE_POLY, a, b, nthreads)


def add_carry(a, b):
    """One instance: (sum limbs, carry-out of the top limb)."""
    a = np.ascontiguousarray(a, dtype=np.uint32).ravel()
    b = np.ascontiguousarray(b, dtype=np.uint32).ravel()
    out = np.empty_like(a)
    c = _load().oracle_add(_p(out), _p(a), _p(b), a.size)
    return out, int(c)


def mul_full_rows(a, b) -> np.ndarray:
    """Per instance (rows) the full 2m-limb product (oracle_mul_full)."""
    a, b = _as2d(a), _as2d(b)
    out = np.empty((a.shape[0], 2 * a.shape[1]), dtype=np.uint32)
    for i in range(a.shape[0]):
        out[i] = mul_full(a[i], b[i])
    return out


def mul_full(a, b) -> np.ndarray:
    """One instance: the full 2m-limb product."""
    a = np.ascontiguousarray(a, dtype=np.uint32).ravel()
    b = np.ascontiguousarray(b, dtype=np.uint32).ravel()
    out = np.empty(2 * a.size, dtype=np.uint32)
    _load().oracle_mul_full(_p(out), _p(a), _p(b), a.size)
    return out
