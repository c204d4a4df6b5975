"""Multi-rank host logic on CPU with the gloo backend, world_size 2 (-m "not gpu").

The GPU path shards instances with no data-path collective;
what can be checked without GPUs is the host side:
* shard ranges partition the batch (weak and strong schemes, ragged n);
* operands generated per rank from global instance indices are bit-identical
  to the single-process batch (so per-rank results equal the N = 1 rows);
* per-rank oracle results gathered over gloo equal the single-process oracle;
* max_over_ranks is the timing reduction bench.py uses.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14642_b200 import inputs, shard


def test_ranges_partition():
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            parts = [shard.strong_range(r, w, n) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    assert [shard.weak_range(r, 4, 10) for r in range(4)] == [(0, 10), (10, 20), (20, 30), (30, 40)]
    with pytest.raises(ValueError):
        shard.strong_range(4, 4, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    lo, hi = shard.strong_range(rank, world, n)
    a, b = inputs.make_operands(hi - lo, m, seed=5, cls="MIX", inst0=lo)
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    res = np.concatenate([O.add(an, bnp), O.mul(an, bnp)], axis=1)
    # gather (plumbing for the test only: the product path has no collective)
    sizes = [shard.strong_range(r, world, n) for r in range(world)]
    t = torch.from_numpy(res.view(np.int32).copy())
    pad = max(h - l for l, h in sizes)
    buf = torch.zeros((pad, 2 * m), dtype=torch.int32)
    buf[: hi - lo] = t
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    tmax = shard.max_over_ranks(float(rank + 1), dist)
    if rank == 0:
        full = torch.cat([bufs[r][: h - l] for r, (l, h) in enumerate(sizes)])
        np.save(os.path.join(out_dir, "gathered.npy"), full.numpy())
        with open(os.path.join(out_dir, "tmax.txt"), "w") as f:
            f.write(str(tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shards_match_single(tmp_path):
    n, m, world = 37, 64, 2
    mp.spawn(_worker, args=(world, _free_port(), n, m, str(tmp_path)), nprocs=world, join=True)
    from oracle import oracle as O
    a, b = inputs.make_operands(n, m, seed=5, cls="MIX")
    an, bnp = inputs.to_numpy_u32(a), inputs.to_numpy_u32(b)
    want = np.concatenate([O.add(an, bnp), O.mul(an, bnp)], axis=1)
    got = np.load(os.path.join(tmp_path, "gathered.npy")).view(np.uint32)
    assert np.array_equal(got, want)
    assert float(open(os.path.join(tmp_path, "tmax.txt")).read()) == float(world)


def test_generator_shard_invariance():
    full_a, full_b = inputs.make_operands(100, 32, seed=3, cls="MIX")
    for (lo, hi) in [(0, 13), (13, 50), (50, 100)]:
        a, b = inputs.make_operands(hi - lo, 32, seed=3, cls="MIX", inst0=lo)
        assert torch.equal(a, full_a[lo:hi]) and torch.equal(b, full_b[lo:hi])


def _torchrun(args, world, timeout=300):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py")] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    import json
    return json.loads(lines[0])


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_dry_run_world2(scaling):
    """bench.py's own rank plumbing under torchrun, world 2, gloo, no GPU:
    shard plan (n = 37, not divisible by 2), per-rank checksums gathered to
    rank 0, max over ranks.  The gathered checksums must equal those of the
    same global rows generated in one process."""
    n, bits = 37, 2048
    line = _torchrun(["--dry-run", "--scaling", scaling, "--n-inst", str(n), "--bits", str(bits),
                      "--cls", "MIX", "--seed", "4"], world=2)
    m = bits // 32
    assert line["n_gpus"] == 2 and line["max_over_ranks"] == 2.0
    ranges = [tuple(p["range"]) for p in line["per_rank"]]
    want_ranges = [shard.plan(r, 2, n, scaling)[:2] for r in range(2)]
    assert ranges == want_ranges
    total = n if scaling == "strong" else 2 * n
    assert line["global_instances"] == total
    a, b = inputs.make_operands(total, m, seed=4, cls="MIX")
    for p in line["per_rank"]:
        lo, hi = p["range"]
        assert p["ck_a"] == shard.checksum(a[lo:hi]) and p["ck_b"] == shard.checksum(b[lo:hi])
    assert line["global_ck_a"] == shard.checksum(a)
    assert line["global_ck_b"] == shard.checksum(b)


def test_checksum_additive():
    a, _ = inputs.make_operands(37, 32, seed=9, cls="U")
    parts = [shard.checksum(a[lo:hi]) for lo, hi in [shard.strong_range(r, 3, 37) for r in range(3)]]
    assert shard.combine_checksums(parts) == shard.checksum(a)
    with pytest.raises(ValueError):
        shard.plan(0, 2, 10, "bogus")
