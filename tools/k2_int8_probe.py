"""A/B probe: int8 tensor-core K2 vs FP64 DMMA K2 on a scaled config; prints
the worst per-block sample difference and the apply times per path."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
w = configs.scaled(name, n) if n != configs.CONFIGS[name].n else configs.CONFIGS[name]
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
rank, over = (w.rank, w.oversample) if w.rank + w.oversample <= 48 else (36, 12)
cap = n <= 65536
reps = {}
for path in ("fp64", "int8", "int8"):
    hp.set_k2_path(path)
    t0 = time.perf_counter()
    rep = hp.compress(op, t, rank=rank, oversample=over, seed=7, capture=cap)
    hp.device_synchronize()
    dt = time.perf_counter() - t0
    ap = sum(p["apply_ms"] for p in rep.report["phases"] if p["phase"] == "h1")
    print(f"{path}: compress {dt:.3f} s, K2 {ap:.1f} ms", flush=True)
    reps[path] = rep
if cap:
    worst = 0.0
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            x, y = reps["fp64"].captured(l, i), reps["int8"].captured(l, i)
            nx = np.linalg.norm(x)
            if nx > 0:
                worst = max(worst, np.linalg.norm(x - y) / nx)
    print(f"worst block rel diff {worst:.3e}")
