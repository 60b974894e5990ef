"""Summarize an ncu launch list (gpu__time_duration.sum per launch) by kernel:
python tools/launch_summary.py gpurun_out/launches.csv [> profiles/...txt]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rows:
    if "Kernel Name" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[hdr["Kernel Name"]]
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("hpeel::", "").replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += float(r[hdr["Metric Value"]].replace(",", "")) * scale[r[hdr["Metric Unit"]]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {v[0]:8d} {v[1]:10.2f} {100 * v[1] / tot:6.1f}%")
print(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f}")
