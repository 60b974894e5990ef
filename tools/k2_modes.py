"""K2 bottleneck probe: compress a config with K2 in full / no-eval / no-DMMA
modes (hp_debug_set_k2_mode bits: 1 skip eval, 2 skip DMMA, 4 force 64-row CTAs).
usage: python tools/k2_modes.py [config] [mode,mode,...] [n (scaled)]"""
import sys
sys.path.insert(0, "/root/repo")
import paper_2205_03406_b200 as hp
from paper_2205_03406_b200 import configs, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
modes = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 0]
w = configs.scaled(name, int(sys.argv[3])) if len(sys.argv) > 3 else configs.CONFIGS[name]
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
for mode in modes:
    _lib.lib().hp_debug_set_k2_mode(mode)
    rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    ph = [p for p in rep.report["phases"] if p["phase"] == "h1"]
    print(mode, "apply_ms %.1f" % sum(p["apply_ms"] for p in ph), [round(float(p["apply_ms"]), 1) for p in ph][:8],
          flush=True)
