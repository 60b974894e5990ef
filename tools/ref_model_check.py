"""Validates bench.py's reference-arm extrapolation where a full oracle run is
feasible: config 3 scaled to N (default 16384) is compressed in full by the
oracle (measured per phase), and the same quantity is predicted the way the
full-size reference arm predicts it (apply rate on a row subset x exact
columns; peel/QR/B per-flop rates calibrated at N = 4096). Prints JSON."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from oracle import cpu_model as M  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
threads = os.cpu_count() or 1
w = configs.scaled(name, n)
pts = w.points(O)
ws = configs.scaled(name, 4096)
cal = M.calibrate(ws, ws.points(O), threads)
tree = O.BoxTree(O.PointCloud(pts), w.leaf)
counts = M.workload_counts(tree, O.adjacency(tree), w.rank, w.oversample)
rate, rows = M.apply_rate(w, pts, w.rank + w.oversample, 10.0, threads)
pred = M.extrapolate(counts, rate, cal)
t0 = time.time()
total, times, rep, _ = M.timed_compress(w, pts, threads)
print(json.dumps({"config": name, "n": n, "threads": threads, "predicted_s": round(pred["total"], 2),
                  "measured_s": round(total, 2), "ratio_pred_over_measured": round(pred["total"] / total, 3),
                  "predicted_phases_s": {k: round(v, 2) for k, v in pred.items()},
                  "measured_phases_s": {k: round(v, 2) for k, v in times.items()},
                  "apply_rows_sampled": rows, "calibration_n": cal["n"]}))
