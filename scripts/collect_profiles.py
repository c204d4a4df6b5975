#!/usr/bin/env python
"""Copy one round-evidence pass (scripts/gpu_round.sh output in gpurun_out/)
into profiles/ under a round tag:

  <tag>_bench.jsonl          the default bench line (e2e + cpu baseline)
  <tag>_sweep.jsonl          per-(op, size) lines of bench.py --sweep
  <tag>_pytest_gpu.log       tail of the GPU test run
  <tag>_launches_4096.csv    ncu launch list of the bench command
  <tag>_launches_4096_summary.json   per-kernel average and share of the step
  <tag>_ncu_full_4096.txt    ncu --set full summaries + executed SASS mix
  ncu_traffic.json           DRAM bytes per launch (bench.py roofline.traffic)

Usage: collect_profiles.py [tag] (default r01)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
KERNELS = ("mul_ntt_kernel", "mul_classical_kernel", "add_kernel")


def json_lines(path):
    out = []
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            try:
                out.append(json.loads(line))
            except ValueError:
                pass
    return out


def write(name, text):
    with open(os.path.join(P, name), "w") as f:
        f.write(text)
    print("wrote profiles/%s" % name)


def main():
    bench = [d for d in json_lines(os.path.join(G, "bench.log")) if "metric" in d]
    if bench:
        write(TAG + "_bench.jsonl", json.dumps(bench[-1]) + "\n")
    sweep = [d for d in json_lines(os.path.join(G, "sweep.log")) if d.get("sweep")]
    if sweep:
        write(TAG + "_sweep.jsonl", "".join(json.dumps(d) + "\n" for d in sweep))
    pt = os.path.join(G, "pytest_gpu.log")
    if os.path.exists(pt):
        write(TAG + "_pytest_gpu.log", "".join(open(pt).readlines()[-3:]))

    lc = os.path.join(G, "launches.csv")
    if os.path.exists(lc):
        raw = open(lc).read()
        write(TAG + "_launches_4096.csv", raw)
        rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
        hdr = rows[0]
        kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        per = collections.defaultdict(list)
        for r in rows[1:]:
            # the step's kernels only (input generation / checksums are torch kernels outside the timed region)
            if len(r) > mv and r[mv] and r[kn].startswith("void bn::"):
                per[r[kn]].append(float(r[mv].replace(",", "")))
        # ns -> us; share of the step over the kernels of the step
        avg = {k: sum(v) / len(v) / 1000.0 for k, v in per.items()}
        tot = sum(avg.values())
        summ = {
            "source": "ncu --metrics gpu__time_duration.sum --clock-control none -c 80 python bench.py "
                      "--no-e2e --no-cpu --no-fused --steps 5 --warmup 3 (4096 bits, 2^20 instances; "
                      "cold-cache, serialised)",
            "kernels": [{"kernel": k, "launches": len(per[k]), "avg_us": round(avg[k], 2),
                         "share_of_step": round(avg[k] / tot, 4)} for k in sorted(avg, key=avg.get)],
        }
        write(TAG + "_launches_4096_summary.json", json.dumps(summ, indent=1) + "\n")

    text, traffic = [], {}
    for k in KERNELS:
        rep = os.path.join(G, "prof_%s_4k.ncu-rep" % k)
        if not os.path.exists(rep):
            continue
        text.append(subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                                   capture_output=True, text=True).stdout)
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        d = dict(zip(rows[0], rows[2]))
        u = dict(zip(rows[0], rows[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = sum(float(d[m].replace(",", "")) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        traffic["%s@4096" % k] = b
    for k in KERNELS:
        rep = os.path.join(G, "prof_%s_4k.ncu-rep" % k)
        if os.path.exists(rep):
            text.append("== executed SASS mix: %s\n" % k + "\n".join(
                subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_mix.py"), rep],
                               capture_output=True, text=True).stdout.splitlines()[:16]) + "\n")
    if text:
        write(TAG + "_ncu_full_4096.txt", "".join(text))
        write("ncu_traffic.json", json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    main()
