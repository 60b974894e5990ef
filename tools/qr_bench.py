"""K4 micro-benchmark and parity probe: batched range finder on synthetic
sample blocks shaped like a workload's levels (rows x r, numerical rank below
r), timed on the device; a few blocks are checked against scipy's pivoted QR.
usage: python tools/qr_bench.py [r] [kmax] [rows:count ...]"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import scipy.linalg as sla
import paper_2205_03406_b200 as hp

r = int(sys.argv[1]) if len(sys.argv) > 1 else 64
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 48
specs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[3:]] or [(4887, 600), (1330, 2000), (273, 8000), (69, 20000)]
rng = np.random.default_rng(0)
for rows, count in specs:
    base = []
    for _ in range(8):
        u = np.linalg.qr(rng.standard_normal((rows, min(rows, r))))[0]
        s = 10.0 ** (-np.arange(min(rows, r)) / 10.0)
        v = np.linalg.qr(rng.standard_normal((r, min(rows, r))))[0]
        base.append((u * s) @ v.T)
    blocks = [base[i % 8] for i in range(count)]
    assert rows * r * count * 8 < 2e9, "keep the host footprint small"
    qs, ranks, ms = hp.debug_qr(blocks, kmax)
    qs2, ranks2, ms2 = hp.debug_qr(blocks, kmax)
    flops = 2.0 * rows * r * r * count
    worst = 0.0
    for i in range(min(count, 8)):
        qr_, rr, piv = sla.qr(blocks[i], mode="economic", pivoting=True)
        d = np.abs(np.diag(rr))
        keep = min(kmax, int(np.sum(d > 1e-14 * d[0])) if d.size else 0)
        assert ranks[i] == keep, (rows, i, ranks[i], keep)
        qa, qb = qs[i][:, :keep], qr_[:, :keep]
        worst = max(worst, np.abs(qa @ (qa.T @ qb) - qb).max() if keep else 0.0)
    print(f"rows {rows:5d} x {r} count {count:6d}: {ms2:8.2f} ms  {flops / ms2 / 1e9:7.3f} TFLOP/s (2mn^2)  span err {worst:.1e}",
          flush=True)
