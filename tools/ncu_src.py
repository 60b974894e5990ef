"""Summarise an `ncu --page source --csv` SASS dump: top instructions by stall
samples and by shared-memory wavefronts, plus per-opcode totals.
usage: python tools/ncu_src.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
col = {n: i for i, n in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]


def f(r, k):
    try:
        return float(r[col[k]] or 0)
    except ValueError:
        return 0.0


tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_w = sum(f(r, "L1 Wavefronts Shared") for r in data)
print("total stall samples %.0f, shared wavefronts %.3g" % (tot_s, tot_w))
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = defaultdict(float)
for r in data:
    for k in stalls:
        agg[k] += f(r, k)
print("stall reasons:", ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot_s) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
ops = defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].split()[1]
    op = op.split(".")[0]
    ops[op][0] += f(r, "Instructions Executed")
    ops[op][1] += f(r, "Warp Stall Sampling (All Samples)")
    ops[op][2] += f(r, "L1 Wavefronts Shared")
print("%-10s %14s %8s %14s" % ("opcode", "warp-insts", "stall%", "smem-wavefr"))
for op, (n, s, w) in sorted(ops.items(), key=lambda x: -x[1][0])[:top]:
    print("%-10s %14.4g %7.1f%% %14.4g" % (op, n, 100 * s / tot_s, w))
print("\ntop instructions by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    top_stall = max(stalls, key=lambda k: f(r, k))
    print("%6.2f%% %-8s %-60s wf=%.3g" % (100 * f(r, "Warp Stall Sampling (All Samples)") / tot_s, top_stall[6:],
                                         r[col["Source"]][:60], f(r, "L1 Wavefronts Shared")))
