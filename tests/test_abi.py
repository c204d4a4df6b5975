"""C-ABI checks that need no GPU (-m "not gpu").

* libbn.so builds for sm_100a, loads, and exports every symbol include/bn.h
  declares; its cubins are sm_100a and contain no CPU fallback entry points.
* Argument validation returns the documented status synchronously, before
  any device access (so these run on a CPU-only host): bad limb_bits,
  unsupported sizes, misalignment, partial aliasing, n_inst == 0.
* The Python binding refuses CPU tensors (no fallback path exists).
"""
import ctypes
import os
import re
import subprocess

import pytest
import torch

import __graft_entry__ as ge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    ge.build()
    from paper_2405_14642_b200 import bn
    return bn.load()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "bn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bn_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert {"bn_add", "bn_mul_classical", "bn_mul_ntt", "bn_prepare", "bn_run_host"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(r"\bT %s$" % n, out, flags=re.M), n


def test_cubin_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_kernels_use_carry_chains(lib):
    """The classical kernel's column update lowers to IMAD.WIDE.U32 with carry."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun",
                           "_ZN2bn20mul_classical_kernelILi7ELi4EEEvPjPKjS3_m", lib._name],
                          capture_output=True, text=True).stdout
    assert "IMAD.WIDE.U32" in sass and "IADD3.X" in sass


vp = ctypes.c_void_p


def _call(lib, name, out, a, b, n, limbs, bits):
    return getattr(lib, name)(vp(out), vp(a), vp(b), n, limbs, bits, None)


OPS = ["bn_add", "bn_mul_classical", "bn_mul_ntt", "bn_add6"]


@pytest.mark.parametrize("op", OPS)
def test_validation_before_launch(lib, op):
    A, B, O = 0x10000, 0x200000, 0x4000000  # fake, aligned, never dereferenced
    assert _call(lib, op, O, A, B, 4, 32, 7) == 1          # limb_bits
    assert _call(lib, op, O, A, B, 4, 0, 32) == 1          # n_limbs == 0
    assert _call(lib, op, O, A, B, 4, 48, 32) == 2         # 1536 bits: not a power of two
    assert _call(lib, op, O, A, B, 4, 16, 32) == 2         # 512 bits: below 1024
    big = 2 if op == "bn_add6" else 0
    assert _call(lib, op, O, A, B, 0, 16384, 32) == big    # 2^19 bits: cluster sizes for add / NTT
    assert _call(lib, op, O, A, B, 4, 65536, 32) == 2      # 2^21 bits: beyond every op
    assert _call(lib, op, O, A, B, 0, 32, 32) == 0         # n_inst == 0: OK, no launch
    assert _call(lib, op, O, A + 4, B, 4, 32, 32) == 3     # misaligned a
    assert _call(lib, op, O + 8, A, B, 4, 32, 32) == 3     # misaligned out
    assert _call(lib, op, 0, A, B, 4, 32, 32) == 1         # NULL
    assert _call(lib, op, A + 16, A, B, 4, 32, 32) == 4    # out partially overlaps a
    assert _call(lib, op, B - 16, A, B, 4, 32, 32) == 4    # out partially overlaps b


def test_u64_size_rules(lib):
    A, B, O = 0x10000, 0x200000, 0x4000000
    # 4096 u64 limbs = 262144 bits: valid size; it would launch, so only check n_inst=0
    assert _call(lib, "bn_add", O, A, B, 0, 4096, 64) == 0
    assert _call(lib, "bn_add", O, A, B, 0, 8192, 64) == 0     # 2^19 bits: cluster size
    assert _call(lib, "bn_add", O, A, B, 0, 32768, 64) == 2


def test_introspection(lib):
    assert lib.bn_max_bits() == 1 << 20 and lib.bn_min_bits() == 1024
    assert [lib.bn_op_max_bits(op) for op in range(8)] == \
        [1 << 20, 1 << 19, 1 << 20, 1 << 18, 1 << 18, 1 << 18, 1 << 18, 1 << 18]
    assert lib.bn_status_string(3).startswith(b"BN_EALIGN")
    for op in range(6):
        assert lib.bn_launches_per_call(op, 4096) == 1
        assert lib.bn_launches_per_call(op, 3000) == 0
    arr = (ctypes.c_uint32 * 3)()
    lib.bn_ntt_primes(arr)
    ps = list(arr)
    assert ps == sorted(ps) and all(2**29 < p < 2**30 and (p - 1) % (1 << 17) == 0 for p in ps)


def test_binding_refuses_cpu_tensors(lib):
    from paper_2405_14642_b200 import bn
    a = torch.zeros((2, 32), dtype=torch.int32)
    with pytest.raises(ValueError):
        bn.add(a, a)
    with pytest.raises(ValueError):
        bn.mul_ntt(a, a)


def test_ntt_primes_are_prime_with_roots(lib):
    """The library's primes: prime (independent Miller-Rabin), and their
    product exceeds the largest exact coefficient m (2^32-1)^2 at the largest
    size, m = 32768 (reading R10); the kernel models use the same primes."""
    from oracle.ntt_ref import is_prime
    from paper_2405_14642_b200 import bn
    ps = bn.ntt_primes()
    assert all(is_prime(p) for p in ps)
    # the largest size is 2^20 bits: m = 32768 limbs
    assert ps[0] * ps[1] * ps[2] > 32768 * (2**32 - 1) ** 2
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "test_kernel_models", os.path.join(os.path.dirname(os.path.abspath(__file__)), "test_kernel_models.py"))
    models = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(models)
    assert ps == models.PRIMES  # the CPU kernel models use the same set


@pytest.mark.parametrize("op", ["bn_poly_classical", "bn_poly_ntt"])
def test_poly_validation_before_launch(lib, op):
    """The fused Poly entry points validate like bn_add before touching a
    device (the workspace is checked after sizing, on the device)."""
    A, B, O, W = 0x10000, 0x200000, 0x4000000, 0x8000000
    f = getattr(lib, op)
    call = lambda o, a, b, n, limbs, bits: f(vp(o), vp(a), vp(b), n, limbs, bits, vp(W), 1 << 20, None)
    assert call(O, A, B, 4, 32, 7) == 1
    assert call(O, A, B, 4, 48, 32) == 2
    assert call(O, A, B, 4, 16384, 32) == 2                 # Poly: one CTA only
    assert call(O, A, B, 0, 32, 32) == 0
    assert call(O, A + 4, B, 4, 32, 32) == 3
    assert call(A + 16, A, B, 4, 32, 32) == 4
    # invalid arguments -> 0 workspace bytes (no device needed)
    assert lib.bn_poly_workspace_bytes(4, 10, 48, 32) == 0
    assert lib.bn_poly_workspace_bytes(0, 10, 32, 32) == 0
    assert lib.bn_poly_workspace_bytes(5, 0, 32, 32) == 0


@pytest.mark.parametrize("op", ["bn_mul_wide_classical", "bn_mul_wide_ntt"])
def test_wide_validation_before_launch(lib, op):
    A, B, O = 0x10000, 0x200000, 0x4000000
    assert _call(lib, op, O, A, B, 4, 32, 7) == 1
    assert _call(lib, op, O, A, B, 4, 48, 32) == 2
    assert _call(lib, op, O, A, B, 0, 32, 32) == 0
    assert _call(lib, op, O + 4, A, B, 4, 32, 32) == 3
    assert _call(lib, op, A, A, B, 4, 32, 32) == 4          # out == a: twice the size, overlaps
    assert _call(lib, op, A - 16, A, B, 4, 32, 32) == 4
    assert _call(lib, op, O, A, B, 4, 16384, 32) == 2       # 512K-bit inputs: wide products stop at 2^18
    assert lib.bn_launches_per_call(7, 262144) == 1 and lib.bn_launches_per_call(6, 262144) == 1
    assert lib.bn_launches_per_call(7, 524288) == 0


def test_build_stamp_tracks_flags():
    """the in-tree library is reused only when the stamp (sources
    + full nvcc command) matches; other flags never count as up to date."""
    from paper_2405_14642_b200 import _build
    _build.build()
    assert _build.up_to_date()
    assert not _build.up_to_date(_build.LIB, extra=("-DBN_SOME_VARIANT=1",))


def test_add_big_validation_before_launch(lib):
    """bn_add_big argument checks return before any launch (no GPU needed)."""
    f = lib.bn_add_big
    A, B, O, W = 0x10000, 0x20000000, 0x40000000, 0x60000000
    m = 1 << 16  # 2^21 bits
    ws = lib.bn_add_big_workspace_bytes(3, m, 32)
    assert ws > 0 and ws % 16 == 0                 # one 32-bit flag per tile + a counter, 16-byte multiple
    assert lib.bn_add_big_workspace_bytes(6, m, 32) >= 2 * ws - 16
    assert lib.bn_add_big_workspace_bytes(0, m, 32) == 0
    assert lib.bn_add_big_workspace_bytes(3, 1 << 12, 32) == 0      # 2^17 bits: below the range
    assert lib.bn_add_big_workspace_bytes(3, 1 << 26, 32) == 0      # 2^31 bits: above
    assert f(O, A, B, 3, 1 << 12, 32, W, ws, None) == 2             # BN_ESIZE
    assert f(O, A, B, 3, 3 << 14, 32, W, ws, None) == 2             # not a power of two
    assert f(O, A, B, 3, m, 16, W, ws, None) == 1                   # limb_bits
    assert f(O, A, B, 0, m, 32, W, ws, None) == 0                   # n_inst == 0: nothing to do
    assert f(O, A, B, 3, m, 32, 0, ws, None) == 1                   # no workspace
    assert f(O, A, B, 3, m, 32, W, ws - 16, None) == 1              # workspace too small
    assert f(O + 4, A, B, 3, m, 32, W, ws, None) == 3               # alignment
    assert f(A + 16, A, B, 3, m, 32, W, ws, None) == 4              # partial overlap
    assert f(O, A, B, 3, m, 32, O + 64, ws, None) == 4              # workspace overlaps out
