"""Build libbn.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Each .cu under csrc/ is compiled in parallel to an object, then linked into
paper_2405_14642_b200/libbn.so.  `-lineinfo` keeps ncu's source page mapped
to our code.

Staleness: a stamp file next to the library (libbn.so.stamp) records the
sha256 of every source / header and of the full nvcc command line; the
library is rebuilt whenever the stamp differs (not by mtime), so a library
built with other flags is never silently reused.

Kernel-variant builds for A/B timing (`python -m paper_2405_14642_b200._build
--variant NAME -DFOO=1 ...`, or BN_NVCC_EXTRA="-DFOO=1") never touch the
in-tree library: they go to ab/libbn_NAME.so (git-ignored) and are loaded
with BN_LIB_PATH.  The shipped geometry is the defaults in csrc/bn_config.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libbn.so")
ROOT = os.path.dirname(HERE)
AB_DIR = os.path.join(ROOT, "ab")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(ROOT, "include", "bn.h"), os.path.abspath(__file__)])


def _stamp(extra) -> str:
    h = hashlib.sha256()
    h.update(json.dumps([NVCC] + ARCH + FLAGS + list(extra)).encode())
    for d in _deps():
        h.update(os.path.relpath(d, ROOT).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def up_to_date(lib: str = LIB, extra=()) -> bool:
    if not os.path.exists(lib) or not os.path.exists(lib + ".stamp"):
        return False
    with open(lib + ".stamp") as f:
        return f.read().strip() == _stamp(extra)


def _compile(src: str, objdir: str, extra, verbose: bool) -> str:
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC] + ARCH + FLAGS + list(extra) + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def _build_to(lib: str, objdir: str, extra, force: bool, verbose: bool) -> str:
    if not force and up_to_date(lib, extra):
        return lib
    os.makedirs(objdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, objdir, extra, verbose), _sources()))
    tmp = lib + ".tmp%d" % os.getpid()
    r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    os.replace(tmp, lib)
    with open(lib + ".stamp", "w") as f:
        f.write(_stamp(extra) + "\n")
    return lib


def build(force: bool = False, verbose: bool = False) -> str:
    """The shipped library (default flags only).  BN_NVCC_EXTRA, if set, is
    routed to a variant build instead of the in-tree library."""
    extra = os.environ.get("BN_NVCC_EXTRA", "").split()
    if extra:
        return build_variant("env", extra, force=force, verbose=verbose)
    return _build_to(LIB, BUILD, (), force, verbose)


def build_variant(name: str, extra, force: bool = False, verbose: bool = False) -> str:
    """A/B build with extra nvcc flags -> ab/libbn_<name>.so (never libbn.so)."""
    os.makedirs(AB_DIR, exist_ok=True)
    return _build_to(os.path.join(AB_DIR, "libbn_%s.so" % name), os.path.join(BUILD, "variant_" + name),
                     tuple(extra), force, verbose)


if __name__ == "__main__":
    argv = sys.argv[1:]
    force, verbose = "--force" in argv, "-v" in argv
    argv = [a for a in argv if a not in ("--force", "-v")]
    if argv and argv[0] == "--variant":
        print(build_variant(argv[1], argv[2:], force=force, verbose=verbose))
    else:
        print(build(force=force, verbose=verbose))
