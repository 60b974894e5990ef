"""The black-box callback boundary (hp_op_callback: the reference's virtual
LinearOperator::apply / apply_adjoint, proj/include/hpeel/linear_operator.hpp:12-24,
called per color as residual_samples does, proj/src/peeling.cpp:165-177):
a numpy DenseOperator passed through the callback reproduces the oracle's
samples at 1e-12 and its factors / dense blocks, with CountingOperator-style
column counts (proj/src/operators.cpp:320-342) and the apply seconds in the
report; errors raised inside the callback surface from compress()."""
import numpy as np
import pytest

import oracle as O
from paper_2205_03406_b200 import configs
from test_gpu_parity import _compare_with_oracle, rel

pytestmark = pytest.mark.gpu


def dense_callback(hp, a):
    return hp.callback_operator(a.shape[0], lambda x, adj: (a.T if adj else a) @ x,
                                symmetric=bool(np.array_equal(a, a.T)))


def test_c1_through_callback_matches_oracle(hp, gpu_available):
    x = np.sort(O.random_cloud(4096, 1, O.mix_seed(7, 0xC1)), axis=0)
    a = O.kernel_matrix("log", x, x, np.eye(4096, dtype=bool))
    op = dense_callback(hp, a)
    rep, orep, _ = _compare_with_oracle(hp, x, 64, op, O.DenseOperator(a), 20, 10, 7)
    rr = rep.report
    leaf_cols = sum(p["forward_cols"] for p in rr["phases"] if p["phase"] == "leaf")
    # every column the driver reports went through the black box, once
    assert op.columns[0] == rr["forward_cols"] and op.columns[1] == rr["adjoint_cols"]
    assert rr["forward_cols"] - leaf_cols == rr["adjoint_cols"] > 0
    assert all(p["apply_ms"] > 0 for p in rr["phases"])
    err = hp.rel_error_power_method(rep, op, 20, O.mix_seed(7, 0xE51))
    oerr = O.rel_error_power_method(orep, O.DenseOperator(a), 20, O.mix_seed(7, 0xE51))
    assert err <= 2.0 * oerr + 1e-15, (err, oerr)


def test_synthetic_fixture_through_callback(hp, gpu_available):
    pts = O.random_cloud(1500, 2, 5)
    ot = O.BoxTree(O.PointCloud(pts), 40)
    truth = O.synth_rank_structured(ot, O.adjacency(ot), 5, 9)
    _compare_with_oracle(hp, pts, 40, dense_callback(hp, truth), O.DenseOperator(truth), 5, 6, 99,
                         exact_ranks=True)


def test_nonsymmetric_callback(hp, gpu_available):
    """apply_adjoint is called for the adjoint samples (A^T != A)."""
    pts = O.equispaced_1d(512)
    ot = O.BoxTree(O.PointCloud(pts), 64)
    sym = O.synth_rank_structured(ot, O.adjacency(ot), 4, 21)
    a = sym + 0.3 * np.triu(sym, 1)  # same admissible ranks, not symmetric
    _compare_with_oracle(hp, pts, 64, dense_callback(hp, a), O.DenseOperator(a), 6, 6, 5)


def test_callback_matches_builtin_kernel(hp, gpu_available):
    """A Python on-the-fly kernel through the callback vs the built-in K2
    kernel operator on scaled config 3: post-peel samples within 1e-12."""
    w = configs.scaled("c3", 4096)
    pts = w.points()
    k = O.kernel_matrix("log", pts, pts, np.eye(len(pts), dtype=bool))
    t = hp.build_tree(pts, w.leaf)
    a = hp.compress(hp.kernel_operator("log", pts), t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    b = hp.compress(dense_callback(hp, k), t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    worst = 0.0
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            worst = max(worst, rel(b.captured(l, i), a.captured(l, i)))
    assert worst <= 1e-12, worst
    for i in range(len(t.dense_pairs())):
        assert rel(b.dense_block(i), a.dense_block(i)) <= 1e-12


def test_callback_sharded_group(hp, gpu_available):
    """The callback black box under the owner-computes group (each rank reads
    back its own rows of each color's product)."""
    pts = O.random_cloud(2000, 2, 8)
    a = O.kernel_matrix("log", pts, pts, np.eye(2000, dtype=bool))
    t = hp.build_tree(pts, 32)
    one = hp.compress(dense_callback(hp, a), t, rank=8, oversample=6, seed=3, capture=True)
    many = hp.compress_group(dense_callback(hp, a), t, 2, rank=8, oversample=6, seed=3, capture=True)
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            for m in many:
                if m.holds(l, i):
                    for x, y in zip(one.block(l, i), m.block(l, i)):
                        assert np.array_equal(x, y)
    for i in range(len(t.dense_pairs())):
        holder = [m for m in many if m.holds(-1, i)]
        assert len(holder) == 1 and np.array_equal(one.dense_block(i), holder[0].dense_block(i))


def test_callback_errors_propagate(hp, gpu_available):
    t = hp.build_tree(O.equispaced_1d(256), 32)

    def bad(x, adj):
        raise KeyError("black box failure")

    with pytest.raises(KeyError):
        hp.compress(hp.callback_operator(256, bad), t, rank=4, oversample=4, seed=1)
    with pytest.raises(ValueError):  # wrong output shape, reported by the binding
        hp.compress(hp.callback_operator(256, lambda x, adj: np.zeros((3, 3))), t, rank=4, oversample=4, seed=1)


@pytest.mark.parametrize("n,leaf", [(512, 64), (4096, 64)])
def test_non_finite_samples_raise_like_reference(hp, gpu_available, n, leaf):
    """A black box that returns NaN: the reference's qr_orthonormal throws
    std::invalid_argument("non-finite matrix in qr") (proj/src/linalg.cpp:59),
    which leaves compress(); K4 reports such blocks and the driver raises the
    same exception (both K4 routes: short blocks at n = 512, tall ones too at
    n = 4096). The oracle raises alike."""
    pts = O.equispaced_1d(n)
    ot = O.BoxTree(O.PointCloud(pts), leaf)
    a = O.synth_rank_structured(ot, O.adjacency(ot), 4, 21)

    def bad(x, adj):
        y = a @ x
        y[n // 3, 0] = np.nan
        return y

    t = hp.build_tree(pts, leaf)
    with pytest.raises(ValueError, match="non-finite matrix in qr"):
        hp.compress(hp.callback_operator(n, bad, symmetric=True), t, rank=4, oversample=6, seed=5)

    class Bad(O.DenseOperator):
        def apply(self, x):
            y = super().apply(x)
            y[n // 3, 0] = np.nan
            return y

    with pytest.raises(ValueError, match="non-finite matrix in qr"):
        O.compress(Bad(a), ot, 4, 6, 5)
