"""Opcode histogram of a cuobjdump -sass listing (optionally of one address range).
usage: python tools/sass_ops.py file.sass [start_hex end_hex]"""
import re
import sys
from collections import Counter

lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62
c = Counter()
for line in open(sys.argv[1]):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if not m:
        continue
    addr = int(m.group(1), 16)
    if not lo <= addr < hi:
        continue
    toks = m.group(2).split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    c[toks[0].split(".")[0]] += 1
for op, n in c.most_common():
    print("%-10s %d" % (op, n))
