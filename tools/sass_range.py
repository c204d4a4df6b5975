#!/usr/bin/env python
"""Print SASS instructions of a cuobjdump -sass dump between two addresses.
Usage: sass_range.py dump.sass 0xLO 0xHI"""
import re
import sys

lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
for line in open(sys.argv[1]):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*/\*", line)
    if m and lo <= int(m.group(1), 16) <= hi:
        print(m.group(2))
