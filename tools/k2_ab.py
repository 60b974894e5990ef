"""A/B check of two K2 modes: compress a scaled config under each and compare
the captured samples and factors (bit-identical expected: same kernel values,
same DMMA order per output element).
usage: python tools/k2_ab.py [config] [n] [modeA] [modeB]"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2205_03406_b200 as hp
from paper_2205_03406_b200 import configs, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
ma, mb = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 4)
w = configs.scaled(name, n)
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
reps = []
for m in (ma, mb):
    _lib.lib().hp_debug_set_k2_mode(m)
    reps.append(hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True))
_lib.lib().hp_debug_set_k2_mode(0)
worst = 0.0
same = True
for l in range(2, t.depth + 1):
    for i in range(len(t.admissible_pairs(l))):
        a, b = reps[0].captured(l, i), reps[1].captured(l, i)
        same &= np.array_equal(a, b)
        worst = max(worst, float(np.abs(a - b).max() / max(np.abs(a).max(), 1e-300)))
print("k2 A/B", name, n, "modes", ma, mb, "bit-identical" if same else "differs", "max rel diff %.3g" % worst)
