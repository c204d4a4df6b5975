#!/usr/bin/env python
"""Benchmark of the hot path: batched add + classical mul + NTT mul on B200.

A *step* is one pass of the whole hot path (bn_add,
bn_mul_classical, bn_mul_ntt) over one batch of synthetic operands.  At
N = 1 the workload is BASELINE.json configs[1]: 4096-bit integers, batch
sized like the paper's sweep (NumBits * NumInsts = 2^32) ->
2^20 instances per GPU.  Under torchrun every rank processes its own 2^20
instances (weak scaling; instances are independent, no collective on the
data path — the only collectives are the timing barrier / max).

Printed (rank 0): one JSON line.
  value       = 2 * instances / step time  [mults/s] (two multiplications per
                instance per step; the add's time is inside the step)
  ops         = per-kernel device time and rate (add GB/s per PAPER.md:929,
                mults/s, Gu32ops/s per PAPER.md:935)
  roofline    = the dominant kernel against its bound
  e2e         = same metric through bn_run_host with pinned HOST buffers
                (H2D of a, b and D2H of the three results inside the timing)
  cpu_baseline= the C oracle on a bounded sample on this host's cores

`--impl reference` times the oracle itself (the CPU reference arm).
`--sweep` additionally prints one line per (op, size) for 1K..256K bits.
The fused NEXT-row workloads (6-Add, Poly with either multiplication) are
timed after the step on the same inputs and reported under "ops" (not in
`value`, which is the §8(a) step); `--no-fused` skips them.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched mults/sec & add GB/s per size (1K-256K bits), 1/2/4/8×B200"
N_SM = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------- work models
def work(bits: int):
    """Algorithmic work per instance."""
    m = bits // 32
    N = 2 * m
    lg = N.bit_length() - 1
    return {
        "add_bytes": 3 * bits // 8,
        "pp": m * (m + 1) // 2,                                  # 32x32 partial products, Eq. 1
        # 3 primes x (3 transforms x non-trivial twiddle products + N pointwise) + CRT:
        # a radix-2 transform has (N/2) log2 N butterflies of which N - 1 use w^0 = 1
        "modmul": 3 * (3 * ((N // 2) * lg - (N - 1)) + N) + 6 * m,
        "u32ops": 300 * m * (m.bit_length() - 1),                # PAPER.md:935 normalisation
    }


# Per-SM per-clock peaks from the measured int-pipe rates (profiles/r01_int_peak.jsonl):
# IMAD.WIDE.U32 issues at 32 lanes/clk/SM (half rate) -> 32 PP/clk/SM for the
# classical column chain; a Shoup modmul needs IMAD.HI (half rate, 2 slots) +
# 2 IMAD = 4 FMA-pipe slots of 64/clk/SM -> 16 modmul/clk/SM.
PP_PER_CLK_SM = 32.0
MODMUL_PER_CLK_SM = 16.0


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
def time_oracle(bits: int, sample: int, steps: int, warmup: int, seed: int, cls: str):
    """The CPU oracle timed as it stands: per step, oracle add + the schoolbook
    product for each of the two multiplication rows, on `sample` instances."""
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
    for _ in range(steps):
        O.add(an, bnp, nthreads=cores)
        O.mul(an, bnp, nthreads=cores)  # classical row
        O.mul(an, bnp, nthreads=cores)  # NTT row: the oracle defines the result (same schoolbook)
    dt = (time.perf_counter() - t0) / steps
    return {"value": 2 * sample / dt, "unit": "mults/s", "cores": cores, "kind": "oracle",
            "sec_per_step": dt,
            "sample": "%d instances x %d bits (%s), per step oracle_add + 2x oracle_mul "
                      "(schoolbook), %d threads" % (sample, bits, cls, cores)}


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
        "ms_per_step": r["sec_per_step"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "configs[1]: %d-bit batch add + classical mul + NTT mul" % args.bits,
                   "bits": args.bits, "instances_per_step": n, "input_class": args.cls},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": "mults/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bits", type=int, default=4096)
    ap.add_argument("--n-inst", type=int, default=0, help="instances per GPU (default 2^32/bits)")
    ap.add_argument("--cls", default="U")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also print per-(op, size) lines")
    ap.add_argument("--no-fused", action="store_true", help="skip the 6-Add / Poly timings")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2405_14642_b200 import bn, inputs, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return shard.max_over_ranks(x, dist if world > 1 else None, dev)

    peaks = load_peaks()
    bits = args.bits
    m = bits // 32
    n = args.n_inst or (1 << 32) // bits
    inst0, _ = shard.weak_range(rank, world, n)  # weak scaling: rank r owns [r n, (r+1) n)
    bn.prepare(local)
    a, b = inputs.make_operands(n, m, seed=args.seed, cls=args.cls, inst0=inst0, device=dev)
    o_add, o_mc, o_mn = torch.empty_like(a), torch.empty_like(a), torch.empty_like(a)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        bn.add(a, b, out=o_add)
        if ev is not None:
            ev[1].record(stream)
        bn.mul_classical(a, b, out=o_mc)
        if ev is not None:
            ev[2].record(stream)
        bn.mul_ntt(a, b, out=o_mn)
        if ev is not None:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # parity guard on the timed configuration: classical == NTT on this rank's
    # whole shard (cheap next to the step)
    if not torch.equal(o_mc, o_mn):
        raise SystemExit("classical and NTT products differ — refusing to report a number")
    # per-rank output checksums (wrapping int64 sums of the add and product
    # shards): rank r's instances are the global range [r n, (r+1) n), so the
    # N = 1 run's checksum must equal rank 0's at every N
    local_ck = [int(o_add.view(torch.int64).sum().item()), int(o_mn.view(torch.int64).sum().item())]
    if world > 1:
        cks = [None] * world
        dist.all_gather_object(cks, local_ck)
    else:
        cks = [local_ck]

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            step(evs[k])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = max_over_ranks(ms_local)
    op_ms = {
        "add": statistics.mean(e[0].elapsed_time(e[1]) for e in evs),
        "mul_classical": statistics.mean(e[1].elapsed_time(e[2]) for e in evs),
        "mul_ntt": statistics.mean(e[2].elapsed_time(e[3]) for e in evs),
    }
    op_ms = {k: max_over_ranks(v) for k, v in op_ms.items()}
    w = work(bits)
    total_inst = n * world
    value = 2 * total_inst / (ms * 1e-3)
    ops = {
        "add": {"ms": op_ms["add"], "GB/s": total_inst * w["add_bytes"] / (op_ms["add"] * 1e-3) / 1e9,
                "adds/s": total_inst / (op_ms["add"] * 1e-3)},
        "mul_classical": {"ms": op_ms["mul_classical"],
                          "mults/s": total_inst / (op_ms["mul_classical"] * 1e-3),
                          "Gu32ops/s": total_inst * w["u32ops"] / (op_ms["mul_classical"] * 1e-3) / 1e9},
        "mul_ntt": {"ms": op_ms["mul_ntt"], "mults/s": total_inst / (op_ms["mul_ntt"] * 1e-3),
                    "Gu32ops/s": total_inst * w["u32ops"] / (op_ms["mul_ntt"] * 1e-3) / 1e9},
    }
    clocks = sampler.result()
    if not args.no_fused:
        ops.update(time_fused(bn, torch, a, b, o_add, stream, args.steps, n, world, w, max_over_ranks,
                              barrier))

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
                "per_unit": "3*(3*((N/2)*log2 N - (N-1)) + N) + 6m modular products per instance "
                            "(N = 2m; non-trivial twiddles, pointwise, CRT); "
                            "peak = 148 SM x 16 modmul/clk (4 FMA-pipe slots each) x sm_max_mhz"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["peak_source"] = peaks["source"] if roof["bound"] == "hbm" else \
        "derived: measured int-pipe rates (profiles/r01_int_peak.jsonl) x sm_max_mhz"
    roof["traffic"] = load_traffic(roof["kernel"], bits)

    line = {
        "metric": METRIC, "value": value, "unit": "mults/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": "configs[1]: %d-bit batch add + classical mul + NTT mul" % bits,
                   "bits": bits, "instances_per_gpu": n, "global_instances": total_inst,
                   "input_class": args.cls, "seed": args.seed,
                   "l2": "inputs larger than L2 (%d MiB per operand per GPU)" % (n * m * 4 >> 20),
                   "parallelism": "instance-sharded x%d, no collective" % world},
        "ops": ops, "roofline": roof, "clocks": clocks,
        "checksums": {"per_rank_add_mul": cks,
                      "note": "wrapping int64 sums of each rank's add / product outputs; "
                              "rank r = global instances [r n, (r+1) n)"},
        "gpu_launches": 3 * args.steps,
    }

    # ---- end to end through the public API with pinned host buffers
    if not args.no_e2e:
        ah = torch.empty((n, m), dtype=torch.int32, pin_memory=True)
        bh = torch.empty((n, m), dtype=torch.int32, pin_memory=True)
        ah.copy_(a)
        bh.copy_(b)
        outs = [torch.empty((n, m), dtype=torch.int32, pin_memory=True) for _ in range(3)]
        names = ["add", "mul_classical", "mul_ntt"]
        bn.run_host(names, ah, bh, outs)  # warm-up (allocates scratch)
        barrier()
        t_e = time.perf_counter()
        for _ in range(args.e2e_steps):
            bn.run_host(names, ah, bh, outs)
        dt = (time.perf_counter() - t_e) / args.e2e_steps
        barrier()
        dt = max_over_ranks(dt)
        if not torch.equal(outs[2][:1024], o_mn[:1024].cpu()):
            raise SystemExit("e2e result differs from the device path")
        line["e2e"] = {"value": 2 * total_inst / dt, "unit": "mults/s", "ms_per_step": dt * 1e3,
                       "h2d_bytes_per_step": 2 * n * m * 4, "d2h_bytes_per_step": 3 * n * m * 4,
                       "api": "bn_run_host (chunked H2D/compute/D2H on two streams)"}
    # ---- oracle on this host's cores (rank 0, N = 1 only)
    if not args.no_cpu and rank == 0 and world == 1:
        s = oracle_sample_size(bits, target_s=0.5)
        r = time_oracle(bits, s, 20, 1, args.seed, args.cls)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if args.sweep:
        sweep(args, bn, inputs, torch, dev, rank, world, peaks, max_over_ranks, barrier)
    if world > 1:
        dist.destroy_process_group()
    return 0


def fused_rates(name: str, ms: float, total_inst: int, w):
    """Rates of the paper's fused workloads: 6-Add in GB/s
    over 3*bits/8 bytes (the footnote's ideal: read a, b, write one result);
    Poly as 4 multiplications (mults/s) and 4x the 1-Mul Gu32ops count."""
    r = {"ms": ms}
    if name.startswith("mul_wide"):
        r["mults/s"] = total_inst / (ms * 1e-3)
    elif name == "add6":
        r["GB/s"] = total_inst * w["add_bytes"] / (ms * 1e-3) / 1e9
        r["add6/s"] = total_inst / (ms * 1e-3)
    else:
        r["poly/s"] = total_inst / (ms * 1e-3)
        r["mults/s"] = 4 * total_inst / (ms * 1e-3)
        r["Gu32ops/s"] = 4 * total_inst * w["u32ops"] / (ms * 1e-3) / 1e9
    return r


def time_fused(bn, torch, a, b, out, stream, steps, n, world, w, max_over_ranks, barrier):
    """NEXT rows (SURVEY §8(f) #1 fused 6-Add / Poly, #2 full products),
    timed after the step on the same inputs:
    each op `steps` times back to back, CUDA events on the launch stream."""
    wide_out = torch.empty((a.shape[0], 2 * a.shape[1]), dtype=a.dtype, device=a.device)
    fns = {"add6": lambda: bn.add6(a, b, out=out),
           "mul_wide_classical": lambda: bn.mul_wide_classical(a, b, out=wide_out)}
    if a.shape[1] * 32 <= 131072:
        fns["mul_wide_ntt"] = lambda: bn.mul_wide_ntt(a, b, out=wide_out)
    for name, f in (("poly_classical", bn.poly_classical), ("poly_ntt", bn.poly_ntt)):
        ws = bn.poly_workspace(name, a)
        fns[name] = (lambda f=f, ws=ws: f(a, b, out=out, workspace=ws))
    res = {}
    for name, f in fns.items():
        for _ in range(2):
            f()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            f()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / steps)
        res[name] = fused_rates(name, ms, n * world, w)
    return res


def load_traffic(kernel: str, bits: int):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of
    the dominant kernel from the committed ncu --set full capture at this
    size (profiles/ncu_traffic.json, key "<kernel>@<bits>"), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("%s@%d" % (kernel, bits))
    except Exception:
        return None


def sweep(args, bn, inputs, torch, dev, rank, world, peaks, max_over_ranks, barrier):
    """Per-(op, size) lines over 1K..256K bits (every op) and 512K / 1M bits
    (add, mul_ntt: thread-block clusters), paper batch 2^32 bits per GPU."""
    for lb in range(10, 21):
        bits = 1 << lb
        m = bits // 32
        n = (1 << 32) // bits
        a, b = inputs.make_operands(n, m, seed=args.seed, cls=args.cls, inst0=rank * n, device=dev)
        o = torch.empty_like(a)
        w = work(bits)
        fns = [("add", bn.add), ("mul_classical", bn.mul_classical), ("mul_ntt", bn.mul_ntt)]
        fns = [(k, f) for k, f in fns if bits <= bn.max_bits(k)]
        if not args.no_fused and bits <= 262144:
            wsc, wsn = bn.poly_workspace("poly_classical", a), bn.poly_workspace("poly_ntt", a)
            wo = torch.empty((n, 2 * m), dtype=a.dtype, device=dev)
            fns += [("mul_wide_classical", lambda x, y, out: bn.mul_wide_classical(x, y, out=wo))]
            if bits <= 131072:
                fns += [("mul_wide_ntt", lambda x, y, out: bn.mul_wide_ntt(x, y, out=wo))]
            fns += [("add6", bn.add6),
                    ("poly_classical", lambda x, y, out: bn.poly_classical(x, y, out=out, workspace=wsc)),
                    ("poly_ntt", lambda x, y, out: bn.poly_ntt(x, y, out=out, workspace=wsn))]
        for name, f in fns:
            slow = name in ("mul_classical", "poly_classical", "mul_wide_classical") and bits > 32768
            reps = 3 if slow else 20
            for _ in range(2):
                f(a, b, out=o)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f(a, b, out=o)
            e1.record()
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1) / reps)
            tot = n * world
            row = {"sweep": True, "op": name, "bits": bits, "instances": tot, "ms": ms, "n_gpus": world}
            if name in ("add6", "poly_classical", "poly_ntt", "mul_wide_classical", "mul_wide_ntt"):
                row.update(fused_rates(name, ms, tot, w))
                if name == "add6":
                    row["frac_hbm"] = row["GB/s"] / world / peaks["hbm_gbs"]
            elif name == "add":
                row["GB/s"] = tot * w["add_bytes"] / (ms * 1e-3) / 1e9
                row["frac_hbm"] = row["GB/s"] / world / peaks["hbm_gbs"]
            else:
                row["mults/s"] = tot / (ms * 1e-3)
                row["Gu32ops/s"] = tot * w["u32ops"] / (ms * 1e-3) / 1e9
                f_ghz = peaks["sm_max_mhz"] / 1e3
                if name == "mul_classical":
                    row["frac_imad_wide"] = (n * w["pp"] / (ms * 1e-3)) / (N_SM * PP_PER_CLK_SM * f_ghz * 1e9)
                else:
                    row["frac_modmul"] = (n * w["modmul"] / (ms * 1e-3)) / (N_SM * MODMUL_PER_CLK_SM * f_ghz * 1e9)
            if rank == 0:
                print(json.dumps(row), flush=True)
        del a, b, o
        if not args.no_fused and bits <= 262144:
            del wo
        torch.cuda.empty_cache()


if __name__ == "__main__":
    sys.exit(main())
