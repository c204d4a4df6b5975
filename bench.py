#!/usr/bin/env python
"""Benchmark of the hot path: batched add + classical mul + NTT mul on B200.

A *step* is one pass of the whole hot path (bn_add,
bn_mul_classical, bn_mul_ntt) over one batch of synthetic operands.  At
N = 1 the workload is BASELINE.json configs[1]: 4096-bit integers, batch
sized like the paper's sweep (NumBits * NumInsts = 2^32) ->
2^20 instances per GPU.  Under torchrun every rank processes its own 2^20
instances (weak scaling, the default) or its floor(r n / W) share of a
global batch (--scaling strong); instances are independent, no collective on
the data path — the only collectives are the timing barrier / max and the
checksum gather.

Printed (rank 0): one JSON line.
  value       = 2 * instances / step time  [mults/s] (two multiplications per
                instance per step; the add's time is inside the step)
  ops         = per-kernel device time (mean and median) and rate of the
                step's three calls (add GB/s per PAPER.md:929, mults/s,
                Gu32ops/s per PAPER.md:935) with their roofline fractions
  per_size    = the metric "per size": every op at 1K..256K bits on the
                paper batch (2^32 bits per operand per GPU), each timed for
                >= 200 ms after 3 warm-ups, with HBM / integer-pipe fractions
                (counts stated there), the C5 256K ONES row
                and the C3 classical/NTT crossover
  roofline    = the step's dominant kernel against its bound, with the ncu
                FMA-heavy / issue / ALU fractions and DRAM traffic from the
                committed capture (profiles/ncu_kernels.json)
  e2e         = same metric through bn_run_host with pinned HOST buffers
                (H2D of a, b and D2H of the three results inside the timing)
  cpu_baseline= the C oracle on a bounded sample on this host's cores

`--impl reference` times the oracle itself (the CPU reference arm).
`--dry-run` exercises the multi-rank plumbing (shard plan, checksum gather,
max over ranks) on the gloo backend without a GPU (tests/test_multi_rank.py).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched mults/sec & add GB/s per size (1K-256K bits), 1/2/4/8×B200"
N_SM = 148
SEEDS = (1, 2, 3)
SIZES = tuple(1 << k for k in range(10, 19))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ---------------------------------------------------------------- work models
def work(bits: int):
    """Algorithmic work per instance (DESIGN.md §6 "Counts")."""
    m = bits // 32
    N = 2 * m
    lg = N.bit_length() - 1
    return {
        "add_bytes": 3 * bits // 8,
        "pp": m * (m + 1) // 2,                                  # 32x32 partial products, Eq. 1
        # builder count: 3 primes x (3 transforms x NON-TRIVIAL twiddle products
        # + N pointwise) + CRT; a radix-2 transform has (N/2) log2 N butterflies
        # of which N - 1 use w^0 = 1 (no multiplication)
        "modmul": 3 * (3 * ((N // 2) * lg - (N - 1)) + N) + 6 * m,
        # survey count: every butterfly counted
        "modmul_all": 3 * (3 * (N // 2) * lg + N) + 3 * N,
        # survey IMAD-multiply equivalents: Shoup twiddle
        # = 3, Montgomery pointwise = 4, Garner ~ 15 per coefficient
        "imad_eq": 3 * (9 * (N // 2) * lg + 4 * N) + 15 * N,
        "u32ops": 300 * m * (m.bit_length() - 1),                # PAPER.md:935 normalisation
    }


# Per-SM per-clock peaks from the measured int-pipe rates (profiles/r01_int_peak.jsonl):
# IMAD 64 lanes/clk/SM; IMAD.WIDE.U32 and IMAD.HI issue at 32 (half rate, 2
# slots) -> 32 PP/clk/SM for the classical column chain (one IMAD.WIDE each);
# a Shoup modmul = IMAD.HI (2 slots) + 2 IMAD = 4 of 64 FMA-pipe slots -> 16
# modmul/clk/SM.
PP_PER_CLK_SM = 32.0
MODMUL_PER_CLK_SM = 16.0
IMAD_PER_CLK_SM = 64.0


def fractions(op: str, bits: int, n: int, ms: float, peaks) -> dict:
    """Roofline fractions of one launch over n instances (per GPU)."""
    w = work(bits)
    s = ms * 1e-3
    f = peaks["sm_max_mhz"] * 1e6 * N_SM
    if op in ("add", "add6"):
        gbs = n * w["add_bytes"] / s / 1e9
        return {"GB/s": gbs, "frac_hbm": gbs / peaks["hbm_gbs"]}
    if op == "mul_classical":
        return {"frac_imad_pipe": n * w["pp"] / s / (f * PP_PER_CLK_SM)}
    if op == "mul_ntt":
        return {"frac_modmul": n * w["modmul"] / s / (f * MODMUL_PER_CLK_SM),
                "frac_modmul_all": n * w["modmul_all"] / s / (f * MODMUL_PER_CLK_SM),
                "frac_imad_eq": n * w["imad_eq"] / s / (f * IMAD_PER_CLK_SM)}
    return {}


class ClockSampler:
    """NVML SM-clock / throttle-reason sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- oracle arm
def time_oracle(bits: int, sample: int, steps: int, warmup: int, seed: int, cls: str, min_seconds: float = 0.0):
    """The CPU oracle timed as it stands: per step, oracle add + the schoolbook
    product for each of the two multiplication rows, on `sample` instances;
    at least `steps` steps and at least `min_seconds` of CPU time."""
    from oracle import oracle as O
    from paper_2405_14642_b200 import inputs
    m = bits // 32
    a, b = inputs.make_operands(sample, m, seed=seed, cls=cls)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    cores = os.cpu_count() or 1
    for _ in range(warmup):
        O.add(an, bnp, nthreads=cores)
        O.mul(an, bnp, nthreads=cores)
    t0 = time.perf_counter()
    done = 0
    while done < steps or time.perf_counter() - t0 < min_seconds:
        O.add(an, bnp, nthreads=cores)
        O.mul(an, bnp, nthreads=cores)  # classical row
        O.mul(an, bnp, nthreads=cores)  # NTT row: the oracle defines the result (same schoolbook)
        done += 1
    total = time.perf_counter() - t0
    steps = done
    dt = total / steps
    return {"value": 2 * sample / dt, "unit": "mults/s", "cores": cores, "kind": "oracle",
            "sec_per_step": dt, "seconds": total, "cpu_model": cpu_model(),
            "sample": "%d instances x %d bits (%s), per step oracle_add + 2x oracle_mul "
                      "(schoolbook), %d threads, %d steps in %.1f s" % (sample, bits, cls, cores, steps, total)}


def oracle_sample_size(bits: int, target_s: float = 0.25) -> int:
    m = bits // 32
    cores = os.cpu_count() or 1
    per_inst = (m * m) * 1.2e-9 * 2 + m * 2e-9  # ~1.2 ns per PP, two products
    return max(4, min(1 << 16, int(target_s * cores / per_inst)))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = oracle_sample_size(args.bits)
    r = time_oracle(args.bits, n, args.steps, args.warmup, args.seed, args.cls)
    line = {
        "metric": METRIC, "value": r["value"], "unit": "mults/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["sec_per_step"] * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "configs[1]: %d-bit batch add + classical mul + NTT mul" % args.bits,
                   "bits": args.bits, "instances_per_step": n, "input_class": args.cls},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")},
        "e2e": {"value": r["value"], "unit": "mults/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- rank plumbing
class Ranks:
    """torch.distributed plumbing of the bench: barrier, max over ranks,
    gather.  backend "nccl" on the GPU box, "gloo" for --dry-run / tests."""

    def __init__(self, backend: str, device=None):
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = dist if self.world > 1 else None
        self.device = device
        if self.world > 1:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=device)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        from paper_2405_14642_b200 import shard
        return shard.max_over_ranks(x, self.dist, self.device)

    def gather(self, obj):
        from paper_2405_14642_b200 import shard
        return shard.gather_objects(obj, self.dist)

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def run_dry(args):
    """Multi-rank plumbing without a GPU: shard plan, input checksums of each
    rank's global rows, checksum gather and max over ranks (gloo)."""
    from paper_2405_14642_b200 import inputs, shard
    rk = Ranks("gloo")
    m = args.bits // 32
    n = args.n_inst or 37
    lo, hi, total = shard.plan(rk.rank, rk.world, n, args.scaling)
    a, b = inputs.make_operands(hi - lo, m, seed=args.seed, cls=args.cls, inst0=lo)
    local = {"rank": rk.rank, "range": [lo, hi], "ck_a": shard.checksum(a), "ck_b": shard.checksum(b)}
    parts = rk.gather(local)
    t = rk.max(float(rk.rank + 1))
    if rk.rank == 0:
        print(json.dumps({"dry_run": True, "scaling": args.scaling, "n_gpus": rk.world, "bits": args.bits,
                          "global_instances": total, "per_rank": parts,
                          "global_ck_a": shard.combine_checksums(p["ck_a"] for p in parts),
                          "global_ck_b": shard.combine_checksums(p["ck_b"] for p in parts),
                          "max_over_ranks": t}), flush=True)
    rk.barrier()
    rk.close()
    return 0


# ---------------------------------------------------------------- timing helpers
def time_op(torch, f, stream, min_ms=200.0, min_reps=3, warmup=3, max_reps=2000, per_rep=None):
    """Warm up, then time back-to-back launches with one CUDA event pair per
    launch on `stream` until >= min_ms and >= min_reps; per_rep(k) (if
    given) picks the k-th launch's inputs.  Returns per-launch ms."""
    call = (lambda k: f(k)) if per_rep else (lambda k: f())
    for k in range(warmup):
        call(k)
    torch.cuda.synchronize()
    # first estimate the launch time to size the event list
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call(0)
    e1.record(stream)
    torch.cuda.synchronize()
    est = max(e0.elapsed_time(e1), 1e-3)
    reps = int(min(max_reps, max(min_reps, min_ms / est + 1)))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record(stream)
    for k in range(reps):
        call(k)
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    return [evs[k].elapsed_time(evs[k + 1]) for k in range(reps)]


def stats(ts):
    return {"ms": statistics.mean(ts), "ms_median": statistics.median(ts), "reps": len(ts),
            "timed_ms": sum(ts)}


def load_ncu(op: str, bits: int):
    """Counters of the committed ncu --set full capture of `op`'s kernel at
    `bits` (profiles/ncu_kernels.json, key "<op>@<bits>"): kernel name, DRAM
    bytes per launch and FMA-heavy / ALU / issue-active percentages, else
    None."""
    p = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    try:
        with open(p) as f:
            return json.load(f).get("%s@%d" % (op, bits))
    except Exception:
        return None


# ---------------------------------------------------------------- per size
def per_size(args, bn, inputs, torch, dev, stream, rk, peaks, shard):
    """Every op at every size 1K..256K on the paper batch (2^32 bits per
    operand per GPU; weak: per rank, strong: split of W x that), three seeds
    rotated across launches, >= 200 ms per (op, size) after 3 warm-ups."""
    out = {}
    sampler = ClockSampler(rk.local)
    t_start = time.perf_counter()
    with sampler:
        for bits in SIZES:
            m = bits // 32
            n_job = (1 << 32) // bits
            lo, hi, total = shard.plan(rk.rank, rk.world, n_job if args.scaling == "weak" else n_job * rk.world,
                                       args.scaling)
            n = hi - lo
            ab = [inputs.make_operands(n, m, seed=s, cls=args.cls, inst0=lo, device=dev) for s in SEEDS]
            o = torch.empty_like(ab[0][0])
            wo = torch.empty((n, 2 * m), dtype=o.dtype, device=dev)
            ws = {k: bn.poly_workspace(k, ab[0][0]) for k in ("poly_classical", "poly_ntt")}
            fns = {
                "add": lambda x, y: bn.add(x, y, out=o),
                "mul_classical": lambda x, y: bn.mul_classical(x, y, out=o),
                "mul_ntt": lambda x, y: bn.mul_ntt(x, y, out=o),
                "add6": lambda x, y: bn.add6(x, y, out=o),
                "poly_classical": lambda x, y: bn.poly_classical(x, y, out=o, workspace=ws["poly_classical"]),
                "poly_ntt": lambda x, y: bn.poly_ntt(x, y, out=o, workspace=ws["poly_ntt"]),
                "mul_wide_classical": lambda x, y: bn.mul_wide_classical(x, y, out=wo),
            }
            if bits <= bn.max_bits("mul_wide_ntt"):
                fns["mul_wide_ntt"] = lambda x, y: bn.mul_wide_ntt(x, y, out=wo)
            row = {"instances": total}
            for name, f in fns.items():
                slow = bits >= 65536 and name in ("mul_classical", "poly_classical", "mul_wide_classical")
                rk.barrier()
                ts = time_op(torch, lambda k, f=f: f(*ab[k % 3]), stream, per_rep=True,
                             min_ms=(100.0 if slow else 200.0), min_reps=(2 if slow else 3),
                             warmup=(1 if slow else 3))
                st = stats(ts)
                st = {k: (rk.max(v) if k in ("ms", "ms_median") else v) for k, v in st.items()}
                r = {"ms": st["ms"], "ms_median": st["ms_median"], "reps": st["reps"]}
                sec = st["ms"] * 1e-3
                if name in ("add", "add6"):
                    r["GB/s"] = total * work(bits)["add_bytes"] / sec / 1e9
                elif name.startswith("poly"):
                    r["mults/s"] = 4 * total / sec
                    r["poly/s"] = total / sec
                else:
                    r["mults/s"] = total / sec
                if name in ("mul_classical", "mul_ntt"):
                    r["Gu32ops/s"] = total * work(bits)["u32ops"] / sec / 1e9
                r.update({k: v for k, v in fractions(name, bits, n, st["ms"], peaks).items()
                          if k != "GB/s"})
                nc = load_ncu(name, bits)
                if nc:  # pipe fractions of the committed ncu capture
                    r["ncu"] = {k: nc[k] for k in ("fmaheavy_pct", "alu_pct", "issue_pct", "dram_bytes") if k in nc}
                row[name] = r
            if "poly_ntt" in row and "mul_ntt" in row:
                # Poly = 4 products but 10 (not 12) transforms per prime (squarings)
                row["poly_ntt"]["vs_4x_mul_ntt"] = row["poly_ntt"]["ms"] / (4 * row["mul_ntt"]["ms"])
            out[str(bits)] = row
            del ab, o, wo, ws
            torch.cuda.empty_cache()
        # C5: 256K-bit worst-case all-ones carry chains (add + NTT mul)
        bits = 262144
        m = bits // 32
        n_job = (1 << 32) // bits
        lo, hi, total = shard.plan(rk.rank, rk.world, n_job if args.scaling == "weak" else n_job * rk.world,
                                   args.scaling)
        a1, _ = inputs.make_operands(hi - lo, m, seed=1, cls="ONES", inst0=lo, device=dev)
        o = torch.empty_like(a1)
        row = {"instances": total, "input_class": "ONES"}
        for name, f in (("add", bn.add), ("mul_ntt", bn.mul_ntt)):
            rk.barrier()
            st = stats(time_op(torch, lambda f=f: f(a1, a1, out=o), stream))
            ms = rk.max(st["ms"])
            r = {"ms": ms, "ms_median": rk.max(st["ms_median"]), "reps": st["reps"]}
            if name == "add":
                r["GB/s"] = total * work(bits)["add_bytes"] / (ms * 1e-3) / 1e9
            else:
                r["mults/s"] = total / (ms * 1e-3)
            r.update({k: v for k, v in fractions(name, bits, hi - lo, ms, peaks).items() if k != "GB/s"})
            row[name] = r
        one = torch.zeros((m,), dtype=torch.int32, device=dev)
        one[0] = 1
        if not torch.equal(o, one.expand(hi - lo, m)):  # (2^B - 1)^2 = 1 mod 2^B on every instance
            raise SystemExit("256K ONES product is not 1 — refusing to report a number")
        row["note"] = ("ONES operands are one repeated word: DRAM traffic of such data can be compressed "
                       "by the memory system, so a frac_hbm above 1 here is not a kernel property")
        out["262144_ONES"] = row
        del a1, o
        torch.cuda.empty_cache()
    # beyond one CTA: thread-block clusters (512K, 1M) and the
    # decoupled look-back add (4M, 64M bits; 64M also on the all-carry RIPPLE class)
    beyond = {}
    for bits, ops_b, cls in ((1 << 19, ("add", "mul_ntt", "add_big"), args.cls),
                             (1 << 20, ("add", "mul_ntt", "add_big"), args.cls),
                             (1 << 22, ("add_big",), args.cls), (1 << 26, ("add_big",), args.cls),
                             (1 << 26, ("add_big",), "RIPPLE")):
        m = bits // 32
        n_job = (1 << 32) // bits
        lo, hi, total = shard.plan(rk.rank, rk.world, n_job if args.scaling == "weak" else n_job * rk.world,
                                   args.scaling)
        x, y = inputs.make_operands(hi - lo, m, seed=1, cls=cls, inst0=lo, device=dev)
        o = torch.empty_like(x)
        wsb = bn.add_big_workspace(x)
        key = str(bits) + ("" if cls == args.cls else "_" + cls)
        row = {"instances": total, "input_class": cls}
        for name in ops_b:
            f = (lambda: bn.add_big(x, y, out=o, workspace=wsb)) if name == "add_big" else \
                (lambda name=name: getattr(bn, name)(x, y, out=o))
            rk.barrier()
            st = stats(time_op(torch, f, stream))
            ms = rk.max(st["ms"])
            r = {"ms": ms, "ms_median": rk.max(st["ms_median"]), "reps": st["reps"]}
            if name in ("add", "add_big"):
                r["GB/s"] = total * work(bits)["add_bytes"] / (ms * 1e-3) / 1e9
                r["frac_hbm"] = r["GB/s"] / rk.world / peaks["hbm_gbs"]
            else:
                r["mults/s"] = total / (ms * 1e-3)
            row[name] = r
        beyond[key] = row
        del x, y, o, wsb
        torch.cuda.empty_cache()
    out["beyond_one_cta"] = beyond
    # C3: classical vs NTT crossover (first size where the NTT product is faster)
    cross = next((b for b in SIZES if out[str(b)]["mul_ntt"]["ms"] < out[str(b)]["mul_classical"]["ms"]), None)
    meta = {"timing": "per (op, size): 3 warm-ups (1 for classical-type ops >= 64K), then back-to-back "
                      "launches with one CUDA event pair each until >= 200 ms (>= 100 ms and >= 2 launches "
                      "for classical-type ops >= 64K); inputs rotate over seeds %s; mean and median, "
                      "max over ranks" % (SEEDS,),
            "batch": "2^32 bits per operand per GPU (PAPER.md:919); inputs > L2 at every size",
            "counts": "DESIGN.md §6: add 3*bits/8 bytes; classical m(m+1)/2 PP at 32 PP/clk/SM; NTT "
                      "frac_modmul = non-trivial modmuls, frac_modmul_all = every butterfly (SURVEY §8(a)), "
                      "both at 16 modmul/clk/SM; frac_imad_eq = SURVEY A.2 IMAD equivalents at 64/clk/SM; "
                      "peaks at sm_max_mhz",
            "clocks": sampler.result(), "seconds": time.perf_counter() - t_start}
    crossover = {"first_bits_ntt_faster": cross,
                 "classical_over_ntt_ms": {str(b): out[str(b)]["mul_classical"]["ms"] / out[str(b)]["mul_ntt"]["ms"]
                                           for b in SIZES}}
    return out, crossover, meta


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bits", type=int, default=4096)
    ap.add_argument("--n-inst", type=int, default=0,
                    help="instances per GPU (weak) or global (strong); default 2^32/bits per GPU")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--cls", default="U")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-per-size", action="store_true", help="skip the per-size block")
    ap.add_argument("--dry-run", action="store_true", help="gloo plumbing check, no GPU")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)

    import torch

    from paper_2405_14642_b200 import bn, inputs, shard

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rk = Ranks("nccl", dev)

    peaks = load_peaks()
    bits = args.bits
    m = bits // 32
    n_arg = args.n_inst or ((1 << 32) // bits) * (1 if args.scaling == "weak" else rk.world)
    lo, hi, total_inst = shard.plan(rk.rank, rk.world, n_arg, args.scaling)
    n = hi - lo
    bn.prepare(local)
    # three seeded batches rotated across steps (seeds 1, 2, 3); each is
    # larger than L2, so every step streams its operands from HBM
    seeds = tuple(args.seed + k for k in range(3))
    batches = [inputs.make_operands(n, m, seed=s, cls=args.cls, inst0=lo, device=dev) for s in seeds]
    o_add = torch.empty_like(batches[0][0])
    o_mc = [torch.empty_like(o_add) for _ in range(3)]
    o_mn = [torch.empty_like(o_add) for _ in range(3)]
    stream = torch.cuda.current_stream(dev)

    def step(k, ev=None):
        a, b = batches[k % 3]
        if ev is not None:
            ev[0].record(stream)
        bn.add(a, b, out=o_add)
        if ev is not None:
            ev[1].record(stream)
        bn.mul_classical(a, b, out=o_mc[k % 3])
        if ev is not None:
            ev[2].record(stream)
        bn.mul_ntt(a, b, out=o_mn[k % 3])
        if ev is not None:
            ev[3].record(stream)

    for k in range(max(args.warmup, 3)):
        step(k)
    torch.cuda.synchronize()
    # parity guard on the timed configuration: classical == NTT on this rank's
    # whole shard for every seed (cheap next to the step)
    for s in range(3):
        if not torch.equal(o_mc[s], o_mn[s]):
            raise SystemExit("classical and NTT products differ — refusing to report a number")
    # per-rank checksums of seed 1's add / product rows: additive over rows,
    # so their sum equals the N = 1 checksum of the same global rows
    bn.add(*batches[0], out=o_add)
    torch.cuda.synchronize()
    local_ck = {"rank": rk.rank, "range": [lo, hi], "add": shard.checksum(o_add), "mul": shard.checksum(o_mn[0])}
    cks = rk.gather(local_ck)

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    rk.barrier()
    torch.cuda.synchronize()
    with sampler:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            step(k, evs[k])
        t1.record(stream)
        torch.cuda.synchronize()
    rk.barrier()
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = rk.max(ms_local)
    per_k = {
        "add": [e[0].elapsed_time(e[1]) for e in evs],
        "mul_classical": [e[1].elapsed_time(e[2]) for e in evs],
        "mul_ntt": [e[2].elapsed_time(e[3]) for e in evs],
    }
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    op_ms = {k: rk.max(statistics.mean(v)) for k, v in per_k.items()}
    op_med = {k: rk.max(statistics.median(v)) for k, v in per_k.items()}
    w = work(bits)
    value = 2 * total_inst / (ms * 1e-3)
    ops = {}
    for k in per_k:
        sec = op_ms[k] * 1e-3
        r = {"ms": op_ms[k], "ms_median": op_med[k]}
        if k == "add":
            r["GB/s"] = total_inst * w["add_bytes"] / sec / 1e9
            r["adds/s"] = total_inst / sec
        else:
            r["mults/s"] = total_inst / sec
            r["Gu32ops/s"] = total_inst * w["u32ops"] / sec / 1e9
        r.update({kk: v for kk, v in fractions(k, bits, n, op_ms[k], peaks).items() if kk != "GB/s"})
        ops[k] = r
    clocks = sampler.result()

    # roofline of the dominant kernel (per-GPU work / per-launch time)
    dom = max(op_ms, key=op_ms.get)
    f_ghz = peaks["sm_max_mhz"] / 1e3
    if dom == "add":
        ach = n * w["add_bytes"] / (op_ms["add"] * 1e-3) / 1e9
        roof = {"kernel": "add_kernel", "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "per_unit": "3*bits/8 bytes per instance (PAPER.md:929)"}
    elif dom == "mul_classical":
        ach = n * w["pp"] / (op_ms["mul_classical"] * 1e-3) / 1e12
        roof = {"kernel": "mul_classical_kernel", "bound": "alu", "achieved": ach,
                "peak": N_SM * PP_PER_CLK_SM * f_ghz / 1e3, "unit": "Tpp/s",
                "per_unit": "m(m+1)/2 32x32 partial products per instance; peak = 148 SM x 32 "
                            "IMAD.WIDE/clk x sm_max_mhz"}
    else:
        ach = n * w["modmul"] / (op_ms["mul_ntt"] * 1e-3) / 1e12
        roof = {"kernel": "mul_ntt_kernel", "bound": "alu", "achieved": ach,
                "peak": N_SM * MODMUL_PER_CLK_SM * f_ghz / 1e3, "unit": "Tmodmul/s",
                "per_unit": "3*(3*((N/2)*log2 N - (N-1)) + N) + 6m non-trivial modular products per "
                            "instance (N = 2m; twiddles, pointwise, CRT); peak = 148 SM x 16 modmul/clk "
                            "(4 FMA-pipe slots each) x sm_max_mhz",
                "frac_modmul_all": ops["mul_ntt"]["frac_modmul_all"],
                "frac_imad_eq": ops["mul_ntt"]["frac_imad_eq"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["peak_source"] = peaks["source"] if roof["bound"] == "hbm" else \
        "derived: measured int-pipe rates (profiles/r01_int_peak.jsonl) x sm_max_mhz"
    nc = load_ncu(dom, bits)
    roof["traffic"] = nc.get("dram_bytes") if nc else None
    if nc:
        roof["ncu"] = {k: nc[k] for k in ("kernel", "fmaheavy_pct", "alu_pct", "issue_pct", "duration_us", "source")
                       if k in nc}
    roof["share_of_step"] = op_ms[dom] / ms

    line = {
        "metric": METRIC, "value": value, "unit": "mults/s", "n_gpus": rk.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": rk.max(statistics.median(step_ms)),
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "configs[1]: %d-bit batch add + classical mul + NTT mul" % bits,
                   "bits": bits, "instances_per_gpu": n, "global_instances": total_inst,
                   "input_class": args.cls, "seeds": list(seeds),
                   "l2": "inputs larger than L2 (%d MiB per operand per GPU), 3 seeded batches rotated"
                         % (n * m * 4 >> 20),
                   "parallelism": "instance-sharded x%d (%s), no collective" % (rk.world, args.scaling)},
        "ops": ops, "roofline": roof, "clocks": clocks,
        "checksums": {"per_rank": cks,
                      "global_add": shard.combine_checksums(c["add"] for c in cks),
                      "global_mul": shard.combine_checksums(c["mul"] for c in cks),
                      "note": "wrapping 64-bit sums of seed-%d add / product rows; additive over rows, "
                              "so global_* equals the N = 1 value for the same global batch" % seeds[0]},
        "gpu_launches": 3 * args.steps,
    }

    # ---- end to end through the public API with pinned host buffers
    if not args.no_e2e:
        a, b = batches[0]
        ah = torch.empty((n, m), dtype=torch.int32, pin_memory=True)
        bh = torch.empty((n, m), dtype=torch.int32, pin_memory=True)
        ah.copy_(a)
        bh.copy_(b)
        outs = [torch.empty((n, m), dtype=torch.int32, pin_memory=True) for _ in range(3)]
        names = ["add", "mul_classical", "mul_ntt"]
        bn.run_host(names, ah, bh, outs)  # warm-up (allocates scratch)
        rk.barrier()
        t_e = time.perf_counter()
        for _ in range(args.e2e_steps):
            bn.run_host(names, ah, bh, outs)
        dt = (time.perf_counter() - t_e) / args.e2e_steps
        rk.barrier()
        dt = rk.max(dt)
        if not torch.equal(outs[2][:1024], o_mn[0][:1024].cpu()):
            raise SystemExit("e2e result differs from the device path")
        line["e2e"] = {"value": 2 * total_inst / dt, "unit": "mults/s", "ms_per_step": dt * 1e3,
                       "h2d_bytes_per_step": 2 * n * m * 4, "d2h_bytes_per_step": 3 * n * m * 4,
                       "api": "bn_run_host (16 MiB chunks, H2D/compute/D2H on three streams)"}
        del ah, bh, outs
    del batches, o_add, o_mc, o_mn
    torch.cuda.empty_cache()

    # ---- the metric per size (every op, 1K..256K bits), C5 ONES row, C3 crossover
    if not args.no_per_size:
        ps, cross, meta = per_size(args, bn, inputs, torch, dev, stream, rk, peaks, shard)
        line["per_size"] = ps
        line["crossover"] = cross
        line["per_size_meta"] = meta

    # ---- oracle on this host's cores (rank 0; other ranks wait at the barrier)
    if not args.no_cpu and rk.rank == 0:
        target = 2.5 if rk.world == 1 else 1.0
        s = oracle_sample_size(bits, target_s=target / 20)
        r = time_oracle(bits, s, 5, 1, args.seed, args.cls, min_seconds=target)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
    rk.barrier()

    if rk.rank == 0:
        print(json.dumps(line), flush=True)
    rk.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
