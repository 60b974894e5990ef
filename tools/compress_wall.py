import sys, time
sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp
from paper_2205_03406_b200 import configs
w = configs.scaled("c4", 262144)
pts = w.points(); t = hp.build_tree(pts, w.leaf); op = hp.kernel_operator(w.kernel, pts, w.param)
for i in range(3):
    t0 = time.perf_counter()
    rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    t1 = time.perf_counter()
    print(f"call {t1-t0:.3f} s, report wall {rep.report['wall_s_total']:.3f} s", flush=True)
    t2 = time.perf_counter(); del rep; t3 = time.perf_counter()
    print(f"  del rep {t3-t2:.3f} s", flush=True)
