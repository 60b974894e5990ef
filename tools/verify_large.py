"""Compress a (scaled) config and measure the final relative error with the
device power method (rel_error_power_method, proj/src/linalg.cpp:206-218):
python tools/verify_large.py <config> <n> [iters]"""
import sys
import time

sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w = configs.scaled(name, n)
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
t0 = time.perf_counter()
rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
hp.device_synchronize()
t1 = time.perf_counter()
err = hp.rel_error_power_method(rep, op, iters, 11)
t2 = time.perf_counter()
st = rep.storage()
print(f"{name} N={n}: compress {t1 - t0:.2f} s (cold), storage {8 * st['total'] / 1e9:.1f} GB, "
      f"relative error (power method, {iters} iterations) {err:.3e}, verifier {t2 - t1:.1f} s")
