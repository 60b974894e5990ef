"""Parity of the sm_100a path (through the C ABI) against the numpy oracle.

Restates the reference's numerical tests (proj/tests/test_peeling.cpp) on the
device path and compares the device's samples, factors and dense blocks with
oracle/ on the same seeded inputs. Tolerances: FP64 samples 1e-12 relative
(north star), reconstruction within 2x of the oracle's error.
"""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def both_trees(hp, pts, leaf):
    return hp.build_tree(pts, leaf), O.BoxTree(O.PointCloud(pts), leaf)


def dense_rel_error(hp, truth, rep):
    got = rep.apply(np.eye(truth.shape[0]))
    return np.linalg.norm(truth - got, 2) / np.linalg.norm(truth, 2)


def test_payload_matches_oracle(hp, gpu_available):
    pts = np.sort(O.random_cloud(4096, 1, O.mix_seed(7, 0xC1)), axis=0)
    t, ot = both_trees(hp, pts, 64)
    for level, r in [(2, 30), (5, 13)]:
        got = hp.debug_payload(t, level, r, 7)
        want = np.zeros_like(got)
        for b in ot.level_boxes(level):
            pts_b = ot.box(b).points
            want[pts_b, :r] = O.payload_gaussian(ot, b, r, 7, level, 0)
            want[pts_b, r:] = O.payload_gaussian(ot, b, r, 7, level, 1)
        assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


def test_operator_apply(hp, gpu_available):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((300, 2))
    a = rng.standard_normal((300, 300))
    op = hp.dense_operator(a)
    assert rel(op.apply(x), a @ x) < 1e-14
    assert rel(op.apply_adjoint(x), a.T @ x) < 1e-14
    pts = rng.random((300, 3))
    for kind, param in [("log", 1.0), ("invdist4pi", 1.0), ("exp", 0.1)]:
        kop = hp.kernel_operator(kind, pts, param)
        same = np.eye(300, dtype=bool) if kind != "exp" else None
        k = O.kernel_matrix(kind, pts, pts, same, param)
        assert rel(kop.apply(x), k @ x) < 1e-13, kind


def test_exact_recovery_1d(hp, gpu_available):
    pts = O.equispaced_1d(512)
    t, ot = both_trees(hp, pts, 64)
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 6, 77)
    rep = hp.compress(hp.dense_operator(truth), t, rank=6, oversample=8, seed=20240601)
    assert dense_rel_error(hp, truth, rep) <= 1e-9


def test_exact_recovery_adaptive_2d(hp, gpu_available):
    pts = O.random_cloud(700, 2, 31)
    t, ot = both_trees(hp, pts, 48)
    assert not t.fully_populated
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 5, 3)
    rep = hp.compress(hp.dense_operator(truth), t, rank=5, oversample=8, seed=20240601)
    assert dense_rel_error(hp, truth, rep) <= 1e-9


def _compare_with_oracle(hp, pts, leaf, op_dev, op_ref, k, p, seed, sample_tol=1e-12,
                         exact_ranks=False, restrict=False, post_relative=True, peeled_tol=None, block_tol=1e-8,
                         strategy="graph"):
    """Samples: the black-box products A Omega of every block (1e-12), the
    post-peel blocks relative to A Omega (1e-12, or `peeled_tol` where the
    peeled part inherits rank choices made at the 1e-14 noise floor) and --
    where the residual is not ~1e2 below A Omega (post_relative) -- relative
    to the residual itself. Factors: U B V^T per block (1e-8 of the block, or of
    1e-4 x the level's largest block for blocks at the noise floor). Dense
    blocks 1e-9. Report counts equal."""
    t, ot = both_trees(hp, pts, leaf)
    rep = hp.compress(op_dev, t, rank=k, oversample=p, seed=seed, capture=True, strategy=strategy)
    cap, leaf_cap, raw_cap = {}, {}, {}
    orep, oreport = O.compress(op_ref, ot, k, p, seed, cap, leaf_cap, restrict=restrict, raw_capture=raw_cap,
                               strategy=strategy)
    # report counts (proj/src/peeling.cpp:478-488)
    got_phases = [(ph["phase"], ph["level"], ph["colors"], ph["forward_cols"], ph["adjoint_cols"])
                  for ph in rep.report["phases"]]
    want_phases = [(ph["phase"], ph["level"], ph["colors"], ph["forward_cols"], ph["adjoint_cols"])
                   for ph in oreport]
    assert got_phases == want_phases
    r = k + p
    worst, worst_raw, worst_scaled, worst_blk, rank_mismatch, nblocks = 0.0, 0.0, 0.0, 0.0, 0, 0
    for level, blocks in cap.items():
        pairs = t.admissible_pairs(level)
        level_max = max(np.linalg.norm(ou @ ob @ ov.T) for ou, ob, ov in orep.levels[level].values())
        for i, (a, b) in enumerate(pairs):
            y_ref, z_ref = blocks[(a, b)]
            y_raw, z_raw = raw_cap[level][(a, b)]
            got = rep.captured(level, i)
            got_raw = rep.captured_raw(level, i)
            worst = max(worst, rel(got[:, :r], y_ref), rel(got[:, r:], z_ref))
            worst_raw = max(worst_raw, rel(got_raw[:, :r], y_raw), rel(got_raw[:, r:], z_raw))
            worst_scaled = max(worst_scaled,
                               np.linalg.norm(got[:, :r] - y_ref) / max(np.linalg.norm(y_raw), 1e-300),
                               np.linalg.norm(got[:, r:] - z_ref) / max(np.linalg.norm(z_raw), 1e-300))
            uu, bb, vv = rep.block(level, i)
            ou, ob, ov = orep.levels[level][(a, b)]
            # ranks decided at the 1e-14 drop threshold sit at the FP64 noise
            # floor and are not pinned (Eigen vs LAPACK differ there too,
            # SURVEY.md 7 hard part 1); U B V^T is what must agree
            du, dv = abs(uu.shape[1] - ou.shape[1]), abs(vv.shape[1] - ov.shape[1])
            rank_mismatch += (du + dv) > 0
            nblocks += 1
            ref = ou @ ob @ ov.T
            scale = max(np.linalg.norm(ref), 1e-4 * level_max, 1e-300)
            worst_blk = max(worst_blk, np.linalg.norm(uu @ bb @ vv.T - ref) / scale)
    print(f"samples rel {worst:.2e} (vs A Omega {worst_scaled:.2e}; unpeeled {worst_raw:.2e}); "
          f"blocks rel {worst_blk:.2e}; rank mismatches {rank_mismatch}/{nblocks}")
    assert worst_raw <= sample_tol, worst_raw
    assert worst_scaled <= (peeled_tol or sample_tol), worst_scaled
    if post_relative:
        assert worst <= sample_tol, worst
    assert worst_blk <= block_tol, worst_blk
    if exact_ranks:
        assert rank_mismatch == 0
    # the representations as operators (H1Rep::apply, hmatrix.cpp:118-130)
    xr = np.random.default_rng(11).standard_normal((t.num_points, 2))
    app = rel(rep.apply(xr), orep.apply(xr))
    print(f"representation apply rel {app:.2e}")
    assert app <= 1e-10, app
    for i, (lam, mu) in enumerate(t.dense_pairs()):
        got = rep.dense_block(i)
        assert rel(got, orep.dense[(lam, mu)]) <= 1e-9
    return rep, orep, ot


def test_samples_and_factors_match_oracle_synthetic(hp, gpu_available):
    pts = O.random_cloud(1500, 2, 5)
    ot = O.BoxTree(O.PointCloud(pts), 40)
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 5, 9)
    _compare_with_oracle(hp, pts, 40, hp.dense_operator(truth), O.DenseOperator(truth), 5, 6, 99,
                         exact_ranks=True)


def test_c1_dense_log_parity(hp, gpu_available):
    """BASELINE config 1 (explicit dense log kernel, N = 4096, m = 64, k = 20,
    p = 10) with the reference's strong admissibility."""
    x = np.sort(O.random_cloud(4096, 1, O.mix_seed(7, 0xC1)), axis=0)
    same = np.eye(4096, dtype=bool)
    a = O.kernel_matrix("log", x, x, same)
    rep, orep, ot = _compare_with_oracle(hp, x, 64, hp.dense_operator(a), O.DenseOperator(a),
                                         20, 10, 7)
    op = hp.dense_operator(a)
    err = hp.rel_error_power_method(rep, op, 20, O.mix_seed(7, 0xE51))
    oerr = O.rel_error_power_method(orep, O.DenseOperator(a), 20, O.mix_seed(7, 0xE51))
    assert err <= 2.0 * oerr + 1e-15, (err, oerr)


def test_leaf_extraction_diagonal(hp, gpu_available):
    """proj/tests/test_peeling.cpp:114-131."""
    pts = O.equispaced_1d(256)
    t = hp.build_tree(pts, 32)
    diag = np.diag(1.0 + 0.01 * np.arange(256))
    rep = hp.compress(hp.dense_operator(diag), t, rank=4, oversample=8, seed=20240601)
    for i, (lam, mu) in enumerate(t.dense_pairs()):
        d = rep.dense_block(i)
        want = diag[np.ix_(t.box_points(lam), t.box_points(mu))]
        assert np.allclose(d, want, rtol=1e-12, atol=1e-12)
    assert dense_rel_error(hp, diag, rep) <= 1e-10


def test_single_leaf_tree(hp, gpu_available):
    """proj/tests/test_peeling.cpp:143-151."""
    t = hp.build_tree(O.equispaced_1d(48), 64)
    truth = O.gaussian_matrix(48, 48, 13)
    rep = hp.compress(hp.dense_operator(truth), t, rank=6, oversample=8, seed=20240601)
    assert rep.num_pairs(-1) == 1
    assert np.max(np.abs(rep.dense_block(0) - truth)) <= 1e-12


def test_unit_leaf_capacity(hp, gpu_available):
    """proj/tests/test_peeling.cpp:133-141."""
    pts = O.equispaced_1d(32)
    t, ot = both_trees(hp, pts, 1)
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 1, 5)
    rep = hp.compress(hp.dense_operator(truth), t, rank=1, oversample=4, seed=20240601)
    assert dense_rel_error(hp, truth, rep) <= 1e-9


def test_matvec_counts_worked_example(hp, gpu_available):
    """proj/tests/test_peeling.cpp:153-182."""
    t, ot = both_trees(hp, O.equispaced_1d(512), 64)
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 4, 21)
    r = 10
    rep = hp.compress(hp.dense_operator(truth), t, rank=4, oversample=6, seed=20240601)
    for ph in rep.report["phases"]:
        if ph["phase"] == "h1" and ph["level"] == 3:
            assert (ph["colors"], ph["forward_cols"], ph["adjoint_cols"]) == (6, 6 * r, 6 * r)
        if ph["phase"] == "leaf":
            assert (ph["colors"], ph["forward_cols"]) == (3, 3 * 64)
    t2, ot2 = both_trees(hp, O.equispaced_1d(1024), 64)
    truth2 = O.synth_rank_structured(ot2, O.adjacency(ot2), 4, 21)
    rep2 = hp.compress(hp.dense_operator(truth2), t2, rank=4, oversample=6, seed=20240601)
    assert rep2.report["forward_cols"] - rep.report["forward_cols"] == 6 * r


@pytest.mark.parametrize("d,per,leaf", [(1, 256, 8), (2, 32, 4)])
def test_fallback_pattern_strategy_matches_oracle(hp, gpu_available, d, per, leaf):
    """compress with ColoringStrategy::kFallbackPattern on fully populated
    trees (proj/src/peeling.cpp:131-153): the report's colors (6^d per level,
    3^d for the leaf probes) and column counts, every sample block, the
    factors and the dense leaves against the oracle run with the same
    strategy."""
    pts = O.uniform_grid_points(per, d) + 1e-3 * (O.random_cloud(per ** d, d, 5) - 0.5) / per
    t = hp.build_tree(pts, leaf)
    assert t.fully_populated
    rep, _, _ = _compare_with_oracle(hp, pts, leaf, hp.kernel_operator("log", pts), O.KernelOperator("log", pts),
                                     6, 6, 99, strategy="fallback-pattern", post_relative=False)
    colors = {(ph["phase"], ph["colors"]) for ph in rep.report["phases"]}
    assert colors == {("h1", 6 ** d), ("leaf", 3 ** d)}
