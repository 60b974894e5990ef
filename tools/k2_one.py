"""One compress of a config with a given K2 mode (for ncu -k sample_apply captures).
usage: python tools/k2_one.py [config] [mode]"""
import sys
sys.path.insert(0, "/root/repo")
import paper_2205_03406_b200 as hp
from paper_2205_03406_b200 import configs, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = configs.CONFIGS[name]
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
_lib.lib().hp_debug_set_k2_mode(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
print("compress ok", rep.report["phases"][5]["apply_ms"])
