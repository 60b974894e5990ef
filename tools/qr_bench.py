"""K4 micro-benchmark and parity probe: batched range finder on synthetic
sample blocks shaped like a workload's levels (rows x r, singular values
10^(-j / decay)), timed on the device; a few blocks are checked against
scipy's pivoted QR (dgeqp3): kept rank, orthonormality of Q, and the
projection residual |Y - Q Q^T Y| / |Y| next to dgeqp3's.
usage: python tools/qr_bench.py [r] [kmax] [rows:count[:decay] ...]   (HP_QR=householder: k_qr2.cu)"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import scipy.linalg as sla
import paper_2205_03406_b200 as hp

r = int(sys.argv[1]) if len(sys.argv) > 1 else 64
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 48
specs = [tuple(float(x) for x in a.split(":")) for a in sys.argv[3:]] or [(4887, 600), (1330, 2000), (273, 8000), (69, 20000)]
rng = np.random.default_rng(0)
for spec in specs:
    rows, count = int(spec[0]), int(spec[1])
    decay = spec[2] if len(spec) > 2 else 10.0
    base = []
    for _ in range(8):
        u = np.linalg.qr(rng.standard_normal((rows, min(rows, r))))[0]
        s = 10.0 ** (-np.arange(min(rows, r)) / decay)
        v = np.linalg.qr(rng.standard_normal((r, min(rows, r))))[0]
        base.append((u * s) @ v.T)
    blocks = [base[i % 8] for i in range(count)]
    assert rows * r * count * 8 < 2e9, "keep the host footprint small"
    qs, ranks, ms = hp.debug_qr(blocks, kmax)
    qs2, ranks2, ms2 = hp.debug_qr(blocks, kmax)
    flops = 2.0 * rows * r * r * count
    orth = res = res_ref = 0.0
    rank_diff = 0
    for i in range(min(count, 8)):
        y = blocks[i]
        qr_, rr, piv = sla.qr(y, mode="economic", pivoting=True)
        d = np.abs(np.diag(rr))
        keep = min(kmax, int(np.sum(d > 1e-14 * d[0])) if d.size else 0)
        rank_diff = max(rank_diff, abs(int(ranks[i]) - keep))
        qa, qb = qs[i][:, :ranks[i]], qr_[:, :keep]
        assert not qs[i][:, ranks[i]:].any()
        orth = max(orth, np.abs(qa.T @ qa - np.eye(qa.shape[1])).max() if qa.size else 0.0)
        ny = np.linalg.norm(y, 2)
        res = max(res, np.linalg.norm(y - qa @ (qa.T @ y), 2) / ny)
        res_ref = max(res_ref, np.linalg.norm(y - qb @ (qb.T @ y), 2) / ny)
    same = all(np.array_equal(a, b) for a, b in zip(qs[:8], qs2[:8]))
    print(f"rows {rows:5d} x {r} k {kmax} decay {decay:4.1f} count {count:6d}: {ms2:8.2f} ms  {flops / ms2 / 1e9:7.3f} TFLOP/s (2mn^2)  "
          f"rank diff {rank_diff}  orth {orth:.1e}  resid {res:.2e} (dgeqp3 {res_ref:.2e})  rerun identical {same}", flush=True)
