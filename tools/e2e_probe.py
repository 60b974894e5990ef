"""Where the end-to-end time of config 3 goes: tree build, operator upload,
compress with streamed export (setup, device phases, tail after the last kernel).
usage: python tools/e2e_probe.py [config] [n]"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = configs.scaled(name, int(sys.argv[2])) if len(sys.argv) > 2 else configs.CONFIGS[name]
pts = w.points()
tree0 = hp.build_tree(pts, w.leaf)
nf, nd = hp.export_sizes(tree0, w.rank, 1, 0)
hf, hd = hp.pinned_empty(nf), hp.pinned_empty(max(nd, 1))
for it in range(3):
    t0 = time.perf_counter()
    tree = hp.build_tree(pts, w.leaf)
    t1 = time.perf_counter()
    op = hp.kernel_operator(w.kernel, pts, w.param)
    t2 = time.perf_counter()
    rep = hp.compress(op, tree, rank=w.rank, oversample=w.oversample, seed=7, export_to=(hf, hd))
    t3 = time.perf_counter()
    hp.device_synchronize()
    t4 = time.perf_counter()
    r = rep.report
    dev = sum(p["wall_ms_total"] for p in r["phases"])
    print(f"iter {it}: tree {t1 - t0:.3f} op {t2 - t1:.3f} compress call {t3 - t2:.3f} (+sync {t4 - t3:.3f}) "
          f"report wall {r['wall_s_total']:.3f} setup_ms {r['setup_ms']:.1f} phase sum {dev:.0f} ms "
          f"d2h {8 * (nf + nd) / 1e9:.2f} GB", flush=True)
    t5 = time.perf_counter()
    rep2 = hp.compress(op, tree, rank=w.rank, oversample=w.oversample, seed=7)
    hp.device_synchronize()
    print(f"        same tree, no export: {time.perf_counter() - t5:.3f} s (report wall {rep2.report['wall_s_total']:.3f}, setup {rep2.report['setup_ms']:.1f})", flush=True)
    del rep, rep2
