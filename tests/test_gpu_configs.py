"""BASELINE configs on the device: scaled-down instances (same generators,
kernels, leaf sizes and ranks) against the oracle, and full-size runs checked
through size-independent properties."""
import numpy as np
import pytest

import oracle as O
from paper_2205_03406_b200 import configs

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def kernel_dense(w, pts):
    same = np.eye(len(pts), dtype=bool) if w.kernel != "exp" else None
    return O.kernel_matrix(w.kernel, pts, pts, same, w.param)


@pytest.mark.parametrize("name,n", [("c2", 8192), ("c3", 8192), ("c4", 8192), ("c5", 4096)])
def test_scaled_config_matches_oracle(hp, gpu_available, name, n):
    w = configs.scaled(name, n)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    ot = O.BoxTree(O.PointCloud(pts), w.leaf)
    a = kernel_dense(w, pts)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    cap = {}
    orep, oreport = O.compress(O.DenseOperator(a), ot, w.rank, w.oversample, 7, cap)
    got = [(p["phase"], p["level"], p["colors"], p["forward_cols"], p["adjoint_cols"])
           for p in rep.report["phases"]]
    want = [(p["phase"], p["level"], p["colors"], p["forward_cols"], p["adjoint_cols"]) for p in oreport]
    assert got == want
    r = w.rank + w.oversample
    worst = 0.0
    for level, blocks in cap.items():
        for i, (al, be) in enumerate(t.admissible_pairs(level)):
            y, z = blocks[(al, be)]
            s = rep.captured(level, i)
            worst = max(worst, rel(s[:, :r], y), rel(s[:, r:], z))
    assert worst <= 1e-12, worst
    # reconstruction: device rep vs oracle rep on a probe block, and errors
    x = O.gaussian_matrix(n, 3, 5)
    ya, yo = rep.apply(x), orep.apply(x)
    ytrue = a @ x
    err, oerr = rel(ya, ytrue), rel(yo, ytrue)
    print(f"{name} n={n}: samples {worst:.2e}, rep error {err:.3e} (oracle {oerr:.3e})")
    assert err <= 2.0 * oerr + 1e-14


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_size_config_error(hp, gpu_available, name):
    """Full BASELINE size on one GPU: relative spectral error of the
    compressed operator against the on-the-fly black box by the power method
    (proj/tools/hpeel_main.cpp:165-166 seeds), and the apply against rows of
    the black box computed directly."""
    w = configs.CONFIGS[name]
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    err = hp.rel_error_power_method(rep, op, 8, hp.mix_seed(7, 0xE51))
    # spot check: a random block of rows of A x (direct on the host) vs rep x
    rng = np.random.default_rng(1)
    x = rng.standard_normal((w.n, 1))
    y = rep.apply(x)
    rows = rng.choice(w.n, 64, replace=False)
    same = (rows[:, None] == np.arange(w.n)[None, :])
    kr = O.kernel_matrix(w.kernel, pts[rows], pts, same, w.param)
    spot = rel(y[rows], kr @ x)
    print(f"{name}: power-method relative error {err:.3e}, row spot check {spot:.3e}")
    assert err < 1e-6 and spot < 1e-6
