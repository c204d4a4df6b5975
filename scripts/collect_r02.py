#!/usr/bin/env python
"""Copy a scripts/gpu_round2.sh pass (gpurun_out/) into profiles/:

  r02_bench.jsonl                 the default bench line
  r02_pytest_gpu.log              tail of pytest -m gpu
  r02_sanitizer.log               the four compute-sanitizer tools, --big
  r02_launches_4096.csv / _summary.json   ncu launch list of the bench step
  r02_ncu_full.txt                ncu --set full summaries of every kernel cited
  r02/raw_*.csv, r02/src_*.csv.gz the raw metric page and the SASS source page
  ncu_kernels.json                per "<op>@<bits>": DRAM bytes, pipe fractions
Usage: collect_r02.py"""
import collections
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
CAPTURES = {  # tag -> op@bits
    "ntt_4k": "mul_ntt@4096", "classical_4k": "mul_classical@4096", "add_4k": "add@4096",
    "ntt_128k": "mul_ntt@131072", "ntt_256k": "mul_ntt@262144", "add6_128k": "add6@131072",
    "add6_256k": "add6@262144", "polyntt_4k": "poly_ntt@4096", "polyntt_256k": "poly_ntt@262144",
    "widentt_256k": "mul_wide_ntt@262144", "addbig_64m": "add_big@67108864",
    "classical_64k": "mul_classical@65536", "ntt_512k": "mul_ntt@524288", "ntt_1m": "mul_ntt@1048576",
}


def main():
    os.makedirs(os.path.join(P, "r02"), exist_ok=True)
    lines = [l for l in open(os.path.join(G, "bench.log")) if l.startswith("{")]
    with open(os.path.join(P, "r02_bench.jsonl"), "w") as f:
        f.write(lines[-1])
    tail = open(os.path.join(G, "pytest_gpu.log")).read().splitlines()[-3:]
    with open(os.path.join(P, "r02_pytest_gpu.log"), "w") as f:
        f.write("python -m pytest tests -m gpu -q (B200, gpurun)\n" + "\n".join(tail) + "\n")
    if os.path.exists(os.path.join(G, "sanitizer.log")):  # compute-sanitizer may be closed on the pool
        shutil.copy(os.path.join(G, "sanitizer.log"), os.path.join(P, "r02_sanitizer.log"))
    # launch list of the bench step
    raw = open(os.path.join(G, "launches.csv")).read()
    body = raw[raw.index('"ID"'):]
    with open(os.path.join(P, "r02_launches_4096.csv"), "w") as f:
        f.write(body)
    per = collections.defaultdict(list)
    for r in csv.DictReader(io.StringIO(body)):
        if r["Metric Name"] == "gpu__time_duration.sum" and any(k in r["Kernel Name"] for k in ("add_kernel", "mul_classical", "mul_ntt")):
            per[r["Kernel Name"]].append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) / len(v) for v in per.values())  # one launch of each kernel = one step
    summ = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none -k regex:add_kernel|mul_classical|mul_ntt -c 24 python bench.py --no-e2e "
                      "--no-cpu --no-per-size --steps 5 --warmup 3 (4096 bits, 2^20 instances; cold-cache, "
                      "serialised: compare shares, not absolute times)",
            "kernels": [{"kernel": k, "launches": len(v), "avg_us": round(sum(v) / len(v), 2),
                         "share_of_step": round(sum(v) / len(v) / tot, 4)} for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))]}
    with open(os.path.join(P, "r02_launches_4096_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    # ncu --set full
    out = []
    specs = []
    for tag, key in CAPTURES.items():
        s = os.path.join(G, "sum_%s.txt" % tag)
        if os.path.exists(s):
            out.append("### %s (%s)\n%s" % (key, tag, open(s).read()))
        for ext in ("raw_%s.csv", "src_%s.csv.gz"):
            src = os.path.join(G, ext % tag)
            if os.path.exists(src):
                shutil.copy(src, os.path.join(P, "r02", os.path.basename(src)))
        specs.append("%s:%s" % (key, os.path.join(P, "r02", "raw_%s.csv" % tag)))
    with open(os.path.join(P, "r02_ncu_full.txt"), "w") as f:
        f.write("ncu --set full --clock-control none --import-source on, one launch each "
                "(scripts/gpu_round2.sh; tools/ncu_summary.py)\n\n" + "\n".join(out))
    kj = os.path.join(P, "ncu_kernels.json")
    if os.path.exists(kj):
        os.remove(kj)
    # per-size counters first (profiles/r02/ncu_sizes, scripts/gpu_ncu_sizes.sh), then the full
    # captures, which take precedence where both exist
    sizes = sorted(glob.glob(os.path.join(P, "r02", "ncu_sizes", "m_*.csv")))
    if sizes:
        subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "ncu_metrics_json.py"), kj] + sizes)
    specs = [sp for sp in specs if os.path.exists(sp.split(":", 1)[1])]
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "ncu_kernels_json.py"), kj] + specs)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
