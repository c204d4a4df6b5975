"""Thin Python binding over libbn.so (include/bn.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only checks tensor metadata, passes ``data_ptr()`` and the current
CUDA stream, and maps status codes to exceptions.  There is NO CPU fallback:
if the extension is missing or no CUDA device is present, calls raise.

Tensors: ``torch.int32``/``torch.uint32`` (u32 limbs) or ``torch.int64``/
``torch.uint64`` (u64 limbs), shape ``[n_inst, n_limbs]``, contiguous, on a
CUDA device.  Bit patterns are the limbs, little-endian.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BN_LIB_PATH: load another build of the same ABI (A/B timing of kernel
# variants); default is the in-tree library built by __graft_entry__.build().
_LIB_PATH = os.environ.get("BN_LIB_PATH") or os.path.join(_HERE, "libbn.so")
_lock = threading.Lock()
_lib = None

SUPPORTED_BITS = tuple(1 << k for k in range(10, 19))  # every op; add / mul_ntt go to 2^20

_STATUS = {0: "BN_OK", 1: "BN_EINVAL", 2: "BN_ESIZE", 3: "BN_EALIGN", 4: "BN_EALIAS",
           5: "BN_ECUDA", 6: "BN_ENODEV"}

OP_ADD, OP_MUL_CLASSICAL, OP_MUL_NTT, OP_ADD6, OP_POLY_CLASSICAL, OP_POLY_NTT = 0, 1, 2, 3, 4, 5
OPS = {"add": OP_ADD, "mul_classical": OP_MUL_CLASSICAL, "mul_ntt": OP_MUL_NTT, "add6": OP_ADD6,
       "poly_classical": OP_POLY_CLASSICAL, "poly_ntt": OP_POLY_NTT, "mul_wide_classical": 6,
       "mul_wide_ntt": 7}


class BnError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        extra = ""
        if status == 5 and _lib is not None:
            extra = " (cudaError %d)" % _lib.bn_cuda_error()
        super().__init__("%s: %s%s" % (where, _STATUS.get(status, str(status)), extra))


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load libbn.so (built by __graft_entry__.build()); raise if missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise ImportError("libbn.so not built at %s — run __graft_entry__.build()" % _LIB_PATH)
            lib = ctypes.CDLL(_LIB_PATH)
            vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
            sig = {
                "bn_add": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_mul_classical": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_mul_ntt": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_add6": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_mul_wide_classical": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_mul_wide_ntt": ([vp, vp, vp, u64, u32, u32, vp], i32),
                "bn_poly_classical": ([vp, vp, vp, u64, u32, u32, vp, u64, vp], i32),
                "bn_poly_ntt": ([vp, vp, vp, u64, u32, u32, vp, u64, vp], i32),
                "bn_poly_workspace_bytes": ([i32, u64, u32, u32], u64),
                "bn_add_big": ([vp, vp, vp, u64, u32, u32, vp, u64, vp], i32),
                "bn_add_big_workspace_bytes": ([u64, u32, u32], u64),
                "bn_prepare": ([i32], i32),
                "bn_run_host": ([ctypes.POINTER(i32), ctypes.POINTER(vp), i32, vp, vp, u64, u32, u32], i32),
                "bn_max_bits": ([], u32),
                "bn_op_max_bits": ([i32], u32),
                "bn_min_bits": ([], u32),
                "bn_cuda_error": ([], i32),
                "bn_status_string": ([i32], ctypes.c_char_p),
                "bn_launches_per_call": ([i32, u32], u32),
                "bn_ntt_primes": ([ctypes.POINTER(u32)], None),
                "bn_debug_ntt_forward": ([vp, u64, u32, i32, ctypes.POINTER(u32), vp], i32),
                "bn_debug_set_grid_cap": ([u32], None),
            }
            for name, (argt, rest) in sig.items():
                # an older build loaded through BN_LIB_PATH may lack newer
                # entry points: those stay unbound and raise when called
                if hasattr(lib, name):
                    f = getattr(lib, name)
                    f.argtypes = argt
                    f.restype = rest
            _lib = lib
    return _lib


def max_bits(op: str = None) -> int:
    """Largest supported size in bits (of `op`, else of any op)."""
    if op is None:
        return int(load().bn_max_bits())
    return int(load().bn_op_max_bits(OPS[op]))


def _limb_bits(t: torch.Tensor) -> int:
    if t.dtype in (torch.int32, torch.uint32):
        return 32
    if t.dtype in (torch.int64, torch.uint64):
        return 64
    raise TypeError("limb tensors must be int32/uint32 or int64/uint64, got %s" % t.dtype)


def _check(a: torch.Tensor, b: torch.Tensor, out):
    if a.dim() != 2 or a.shape != b.shape:
        raise ValueError("a and b must be [n_inst, n_limbs] with equal shapes")
    if a.dtype != b.dtype:
        raise TypeError("a and b must have the same dtype")
    if not (a.is_cuda and b.is_cuda):
        raise ValueError("operands must be CUDA tensors (no CPU fallback)")
    if a.device != b.device:
        raise ValueError("operands on different devices")
    if not (a.is_contiguous() and b.is_contiguous()):
        raise ValueError("operands must be contiguous")
    if out is None:
        out = torch.empty_like(a)
    elif out.shape != a.shape or out.dtype != a.dtype or out.device != a.device or not out.is_contiguous():
        raise ValueError("out must match a in shape, dtype, device and be contiguous")
    return out


class _on_device:
    """Make `dev` the current CUDA device for a C-ABI call (the library
    launches on the current device) — a no-op when it already is, which
    keeps the per-call host cost low for small batches."""

    __slots__ = ("dev", "prev")

    def __init__(self, dev: torch.device):
        self.dev = dev.index

    def __enter__(self):
        self.prev = torch.cuda.current_device()
        if self.prev != self.dev:
            torch.cuda.set_device(self.dev)
        return torch._C._cuda_getCurrentRawStream(self.dev)

    def __exit__(self, *exc):
        if self.prev != self.dev:
            torch.cuda.set_device(self.prev)


def _call(name: str, a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    out = _check(a, b, out)
    lib = _lib if _lib is not None else load()
    n_inst, n_limbs = a.shape
    with _on_device(a.device) as stream:
        st = getattr(lib, name)(out.data_ptr(), a.data_ptr(), b.data_ptr(), n_inst, n_limbs,
                                _limb_bits(a), stream)
    if st != 0:
        raise BnError(st, name)
    return out


def add(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """(a + b) mod 2^bits per instance (bn_add)."""
    return _call("bn_add", a, b, out)


def mul_classical(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """(a * b) mod 2^bits per instance, quadratic algorithm (bn_mul_classical)."""
    return _call("bn_mul_classical", a, b, out)


def mul_ntt(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """(a * b) mod 2^bits per instance, exact 3-prime NTT (bn_mul_ntt)."""
    return _call("bn_mul_ntt", a, b, out)


def _wide(name: str, a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    _check(a, b, a)  # operand checks only
    n_inst, n_limbs = a.shape
    if out is None:
        out = torch.empty((n_inst, 2 * n_limbs), dtype=a.dtype, device=a.device)
    elif out.shape != (n_inst, 2 * n_limbs) or out.dtype != a.dtype or out.device != a.device \
            or not out.is_contiguous():
        raise ValueError("out must be [n_inst, 2*n_limbs], a's dtype and device, contiguous")
    lib = load()
    with _on_device(a.device) as stream:
        st = getattr(lib, name)(out.data_ptr(), a.data_ptr(), b.data_ptr(), n_inst, n_limbs,
                                _limb_bits(a), stream)
    if st != 0:
        raise BnError(st, name)
    return out


def mul_wide_classical(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """Full product a * b (2 n_limbs limbs per instance), quadratic algorithm."""
    return _wide("bn_mul_wide_classical", a, b, out)


def mul_wide_ntt(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """Full product a * b (2 n_limbs limbs per instance), exact NTT; bits <= 262144."""
    return _wide("bn_mul_wide_ntt", a, b, out)


ADD_BIG_MIN_BITS, ADD_BIG_MAX_BITS = 1 << 18, 1 << 30


def add_big_workspace(a: torch.Tensor) -> torch.Tensor:
    """A workspace tensor for add_big on a's device (tile flags + counter)."""
    nb = int(load().bn_add_big_workspace_bytes(a.shape[0], a.shape[1], _limb_bits(a)))
    return torch.empty(max(16, nb), dtype=torch.uint8, device=a.device)


def add_big(a: torch.Tensor, b: torch.Tensor, out=None, workspace=None) -> torch.Tensor:
    """(a + b) mod 2^bits for 2^18 .. 2^30-bit instances, decoupled look-back
    carry scan over 2^18-bit tiles (bn_add_big)."""
    out = _check(a, b, out)
    if workspace is None:
        workspace = add_big_workspace(a)
    if not workspace.is_cuda or workspace.device != a.device or not workspace.is_contiguous():
        raise ValueError("workspace must be a contiguous CUDA tensor on the operands' device")
    lib = load()
    n_inst, n_limbs = a.shape
    with _on_device(a.device) as stream:
        st = lib.bn_add_big(out.data_ptr(), a.data_ptr(), b.data_ptr(), n_inst, n_limbs, _limb_bits(a),
                            workspace.data_ptr(), workspace.numel() * workspace.element_size(), stream)
    if st != 0:
        raise BnError(st, "bn_add_big")
    return out


def add6(a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
    """6-Add: (4a + 3b) mod 2^bits as six fused scan-additions (bn_add6)."""
    return _call("bn_add6", a, b, out)


def poly_workspace_bytes(op: str, n_inst: int, n_limbs: int, limb_bits: int = 32) -> int:
    """Workspace bytes bn_poly_* needs on the current device."""
    return int(load().bn_poly_workspace_bytes(OPS[op], n_inst, n_limbs, limb_bits))


def poly_workspace(op: str, a: torch.Tensor) -> torch.Tensor:
    """A workspace tensor for poly_* on a's device (reusable across calls on one stream)."""
    with torch.cuda.device(a.device):
        nb = poly_workspace_bytes(op, a.shape[0], a.shape[1], _limb_bits(a))
    return torch.empty(max(16, nb), dtype=torch.uint8, device=a.device)


def _poly(name: str, op: str, a, b, out, workspace):
    out = _check(a, b, out)
    if workspace is None:
        workspace = poly_workspace(op, a)
    if not workspace.is_cuda or workspace.device != a.device or not workspace.is_contiguous():
        raise ValueError("workspace must be a contiguous CUDA tensor on the operands' device")
    lib = load()
    n_inst, n_limbs = a.shape
    with _on_device(a.device) as stream:
        st = getattr(lib, name)(out.data_ptr(), a.data_ptr(), b.data_ptr(), n_inst, n_limbs, _limb_bits(a),
                                workspace.data_ptr(), workspace.numel() * workspace.element_size(), stream)
    if st != 0:
        raise BnError(st, name)
    return out


def poly_classical(a: torch.Tensor, b: torch.Tensor, out=None, workspace=None) -> torch.Tensor:
    """Poly: ((a a + b)(b b + b) + a b) mod 2^bits, classical products, one kernel."""
    return _poly("bn_poly_classical", "poly_classical", a, b, out, workspace)


def poly_ntt(a: torch.Tensor, b: torch.Tensor, out=None, workspace=None) -> torch.Tensor:
    """Poly: ((a a + b)(b b + b) + a b) mod 2^bits, NTT products, one kernel."""
    return _poly("bn_poly_ntt", "poly_ntt", a, b, out, workspace)


def prepare(device: int = 0) -> None:
    st = load().bn_prepare(device)
    if st != 0:
        raise BnError(st, "bn_prepare")


def run_host(ops, a: torch.Tensor, b: torch.Tensor, outs=None):
    """End-to-end path over HOST tensors (ideally pinned): bn_run_host.
    ``ops`` is a list of names from OPS; returns the list of host outputs."""
    if a.is_cuda or b.is_cuda:
        raise ValueError("run_host takes host tensors")
    if a.dim() != 2 or a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError("a and b must be [n_inst, n_limbs] with equal shapes and dtypes")
    if not (a.is_contiguous() and b.is_contiguous()):
        raise ValueError("operands must be contiguous")
    codes = [OPS[o] for o in ops]
    if outs is None:
        outs = [torch.empty_like(a, pin_memory=a.is_pinned()) for _ in codes]
    lib = load()
    n = len(codes)
    c_ops = (ctypes.c_int * n)(*codes)
    c_outs = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
    st = lib.bn_run_host(c_ops, c_outs, n, a.data_ptr(), b.data_ptr(), a.shape[0], a.shape[1],
                         _limb_bits(a))
    if st != 0:
        raise BnError(st, "bn_run_host")
    return outs


def ntt_primes():
    arr = (ctypes.c_uint32 * 3)()
    load().bn_ntt_primes(arr)
    return [int(x) for x in arr]


def debug_ntt_forward(x: torch.Tensor, prime: int):
    """Forward NTT of each row of x (int32 residues, length N = 2^lg), in place,
    bit-reversed output; returns (x, omega).  Test/debug entry point only."""
    if x.dim() != 2 or not x.is_cuda or not x.is_contiguous() or x.dtype not in (torch.int32, torch.uint32):
        raise ValueError("x must be a contiguous CUDA int32 [n, N] tensor")
    n, N = x.shape
    lg = N.bit_length() - 1
    if 1 << lg != N:
        raise ValueError("N must be a power of two")
    om = ctypes.c_uint32()
    with torch.cuda.device(x.device):
        st = load().bn_debug_ntt_forward(x.data_ptr(), n, lg, prime, ctypes.byref(om),
                                         torch.cuda.current_stream(x.device).cuda_stream)
    if st != 0:
        raise BnError(st, "bn_debug_ntt_forward")
    return x, int(om.value)


def debug_set_grid_cap(cap: int) -> None:
    """Tests only: cap every kernel's grid (0 = default)."""
    load().bn_debug_set_grid_cap(int(cap))


def launches_per_call(op: str, bits: int) -> int:
    return int(load().bn_launches_per_call(OPS[op], bits))
