"""One compress of a (scaled) BASELINE config, for ncu captures:
python tools/one_compress.py <config> <n> [fp64|int8]"""
import sys

sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
if len(sys.argv) > 3:
    hp.set_k2_path(sys.argv[3])
w = configs.scaled(name, n)
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
hp.device_synchronize()
print("ok", round(rep.report["wall_s_total"], 3), [(p["level"], round(p["apply_ms"], 1), round(p["peel_ms"], 1),
                                                    round(p["qr_ms"], 1), round(p["bsolve_ms"], 1))
                                                   for p in rep.report["phases"]])
