#!/usr/bin/env python
"""Build an A/B variant library (ab/libbn_NAME.so) and print registers /
spills of the kernels whose mangled name contains PATTERN.
Usage: variant_build.py NAME PATTERN [-DFOO=1 ...]"""
import os
import re
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, pat, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
r = subprocess.run([sys.executable, "-m", "paper_2405_14642_b200._build", "--variant", name, "--force", "-v"] + flags,
                   capture_output=True, text=True, cwd=root)
if r.returncode:
    sys.exit(r.stderr[-3000:])
cur, spill = None, None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = m.group(0)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat in cur:
        print("%-8s %-50s regs %s, %s" % (name, cur[:50], m.group(1), spill))
print(r.stdout.strip())
