"""Kernel-level parity probes of the sm_100a path through the C ABI."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_log_accuracy(hp, gpu_available):
    """The log-kernel black box evaluates log on the device with its own
    argument reduction (device.cuh fast_log); <= 2 ulp against libm."""
    rng = np.random.default_rng(0)
    x = np.concatenate([
        np.exp(rng.uniform(-700, 700, 200000)),
        1.0 + rng.uniform(-1e-3, 1e-3, 50000),
        rng.uniform(0.5, 2.0, 50000),
        np.array([1.0, 2.0, 0.5, math.sqrt(2.0), math.sqrt(0.5), 1e-300, 1e300, 3.0]),
    ])
    got = hp.debug_log(x)
    want = np.array([math.log(v) for v in x])
    ulp = np.spacing(np.abs(want))
    err = np.abs(got - want)
    # absolute bound near x = 1 (log -> 0), 2 ulp elsewhere
    assert np.all(err <= np.maximum(2.0 * ulp, 2.2e-16 * np.abs(x - 1.0) + 1e-300))


def _spectrum_block(rng, rows, r, decay):
    q = min(rows, r)
    u = np.linalg.qr(rng.standard_normal((rows, q)))[0]
    v = np.linalg.qr(rng.standard_normal((r, q)))[0]
    return (u * 10.0 ** (-np.arange(q) / decay)) @ v.T


@pytest.mark.parametrize("r,kmax", [(42, 32), (64, 48), (80, 64), (14, 6), (96, 96), (96, 64), (33, 33), (8, 3)])
def test_range_finder_matches_pivoted_qr(hp, gpu_available, r, kmax):
    """K4 (k_gqr.cu: staged pivoted Cholesky-QR) against LAPACK's dgeqp3 on
    ragged batches: kept rank (|R_jj| > 1e-14 |R_00|, capped at kmax,
    proj/src/linalg.cpp:53-78), orthonormal Q, zero columns beyond the rank
    and the projection residual |Y - Q Q^T Y|, which equals dgeqp3's when the
    same columns are chosen. Spectra from one stage (decay 10) to three
    (decay 1.5), short (rows < r), tall (row tasks + partial Gram sums),
    exactly rank-deficient and zero blocks."""
    import scipy.linalg as sla

    rng = np.random.default_rng(r)
    blocks = []
    for rows, decay in [(256, 10.0), (128, 3.0), (100, 1.5), (33, 4.0), (7, 2.0), (1500, 5.0), (600, 2.0)]:
        for _ in range(3):
            blocks.append(_spectrum_block(rng, rows, r, decay))
    blocks += [_spectrum_block(rng, 1, r, 3.0), _spectrum_block(rng, 2, r, 3.0), _spectrum_block(rng, 257, r, 6.0)]
    low = rng.standard_normal((90, 5)) @ rng.standard_normal((5, r))  # exact rank 5
    blocks += [low, np.zeros((40, r)), 1e-200 * _spectrum_block(rng, 64, r, 3.0)]
    qs, ranks, _ = hp.debug_qr(blocks, kmax)
    qs2, ranks2, _ = hp.debug_qr(blocks, kmax)
    for y, q, keep, q2 in zip(blocks, qs, ranks, qs2):
        qr_, rr, _ = sla.qr(y, mode="economic", pivoting=True)
        d = np.abs(np.diag(rr))
        want = min(kmax, int(np.sum(d > 1e-14 * d[0]))) if d.size and d[0] > 0 else 0
        # the keep rule sits at the FP64 noise floor for the deepest spectra
        assert abs(int(keep) - want) <= (1 if want < min(kmax, min(y.shape)) else 0), (y.shape, keep, want)
        assert np.array_equal(q, q2)  # run-to-run identical
        assert not q[:, keep:].any()
        qa = q[:, :keep]
        assert np.abs(qa.T @ qa - np.eye(keep)).max() <= 1e-13 if keep else True
        ny = np.linalg.norm(y, 2)
        if ny == 0.0 or keep != want:
            continue
        res = np.linalg.norm(y - qa @ (qa.T @ y), 2) / ny
        ref = np.linalg.norm(y - qr_[:, :want] @ (qr_[:, :want].T @ y), 2) / ny
        assert res <= 1.05 * ref + 1e-14, (y.shape, res, ref)
