#!/usr/bin/env python
"""Registers / spills per kernel from a verbose (-Xptxas -v) rebuild of libbn.so."""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, "-c", "from paper_2405_14642_b200 import _build; "
                      "_build.build(force=True, verbose=True)"], capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur).replace("void ", "")
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print("%-45s regs %3s spill st/ld %s" % (cur, m.group(1), spill))
        cur = None
