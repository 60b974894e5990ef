"""One compress of scaled c3 on the int8 K2 path (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
if len(sys.argv) > 2:
    hp.set_k2_path(sys.argv[2])
w = configs.scaled("c3", n)
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
hp.device_synchronize()
print("ok", [round(p["apply_ms"], 2) for p in rep.report["phases"]])
