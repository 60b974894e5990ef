"""Pins the CPU oracle against the reference's own known-answer and tolerance
tests (the reference ships no golden data). Each test cites the
reference test it restates."""
import math

import numpy as np
import pytest

import oracle as O


def tree_of(pts, leaf):
    t = O.BoxTree(O.PointCloud(pts), leaf)
    return t, O.adjacency(t)


def box_at(t, level, coord):
    for b in t.level_boxes(level):
        if t.box(b).coord[0] == coord:
            return b
    raise AssertionError


# ---------------------------------------------------------------- RNG
def test_gaussian_stream_frozen():
    """proj/include/hpeel/rng.hpp:12-17, :44-48: vectorized stream equals the
    scalar libm stream; determinism and moments (test_linalg.cpp:23-41)."""
    for rows, cols, seed in [(4, 3, 7), (5, 7, 9), (1, 1, 0), (13, 5, 2**63 + 5)]:
        a = O.gaussian_matrix(rows, cols, seed)
        b = O.gaussian_matrix_libm(rows, cols, seed)
        assert np.max(np.abs(a - b)) <= 4e-16 * max(1.0, np.max(np.abs(b)))
    g = O.gaussian_matrix(400, 250, 12345)
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1.0) < 0.01
    st = O.SplitMix64(42)
    first = [st.next() for _ in range(3)]
    assert first[0] == O.scramble((42 + O.GAMMA) % 2**64)
    assert O.mix_seed(5, 1, 2) == O.mix_seed(O.mix_seed(5, 1), 2)


def test_random_cloud_stream():
    """proj/src/operators.cpp:88-95: row-major next_closed_open."""
    pts = O.random_cloud(5, 3, 99)
    st = O.SplitMix64(99)
    want = np.array([[st.next_closed_open() for _ in range(3)] for _ in range(5)])
    assert np.array_equal(pts, want)


# ---------------------------------------------------------------- tree
def test_figure_tree():
    """proj/tests/test_box_tree.cpp:30-41."""
    t, _ = tree_of(O.equispaced_1d(400), 100)
    assert t.depth == 2
    assert len(t.box(0).points) == 400
    assert len(t.level_boxes(1)) == 2 and len(t.box(t.level_boxes(1)[0]).points) == 200
    assert len(t.level_boxes(2)) == 4 and len(t.box(t.level_boxes(2)[0]).points) == 100
    assert list(t.box(t.level_boxes(1)[0]).points) == list(range(200))


def test_single_point_and_partition():
    """proj/tests/test_box_tree.cpp:43-62."""
    t, _ = tree_of(np.array([[0.3, 0.4]]), 10)
    assert t.depth == 0 and t.num_boxes == 1 and t.box(0).is_leaf
    t, _ = tree_of(O.random_cloud(1000, 2, 99), 50)
    seen = np.zeros(1000, dtype=int)
    for b in t.boxes:
        if b.is_leaf:
            assert len(b.points) <= 50
            seen[b.points] += 1
    assert np.all(seen == 1)


def test_coincident_points_fail():
    """proj/tests/test_box_tree.cpp:64-68."""
    with pytest.raises(RuntimeError):
        O.BoxTree(O.PointCloud(np.zeros((10, 1))), 2)


def test_doubling_adds_a_level():
    """proj/tests/test_box_tree.cpp:81-88."""
    prev = O.BoxTree(O.PointCloud(O.equispaced_1d(256)), 32).depth
    for n in (512, 1024, 2048, 4096):
        d = O.BoxTree(O.PointCloud(O.equispaced_1d(n)), 32).depth
        assert d == prev + 1
        prev = d


def test_worked_example_lists_and_pairs():
    """proj/tests/test_box_tree.cpp:90-117."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    assert t.depth == 3
    b4, b5, b6, b7 = (box_at(t, 2, c) for c in range(4))
    assert adj.neighbors[b4] == [b4, b5]
    assert adj.interaction[b4] == [b6, b7]
    assert adj.interaction[b7] == [b4, b5]
    assert adj.neighbors[0] == [0] and adj.interaction[0] == []
    assert len(O.admissible_pairs(t, adj, 2)) == 6
    pairs = O.admissible_pairs(t, adj, 3)
    assert len(pairs) == 18
    assert all((b, a) in set(pairs) for a, b in pairs)


@pytest.mark.parametrize("d,max_n,max_i", [(2, 9, 27), (3, 27, 189)])
def test_uniform_grid_limits(d, max_n, max_i):
    """proj/tests/test_box_tree.cpp:119-148."""
    t, adj = tree_of(O.uniform_grid_points(8, d), 1)
    assert t.depth == 3
    assert max(len(adj.neighbors[b]) for b in t.level_boxes(3)) == max_n
    assert max(len(adj.interaction[b]) for b in t.level_boxes(3)) == max_i


def test_adjacency_symmetry_and_dense_pairs():
    """proj/tests/test_box_tree.cpp:150-187."""
    t, adj = tree_of(O.random_cloud(600, 2, 17), 40)
    for b in t.boxes:
        for n in adj.neighbors[b.id]:
            assert b.id in adj.neighbors[n]
        for i in adj.interaction[b.id]:
            assert b.id in adj.interaction[i] and t.box(i).level == b.level
    raw = np.concatenate([0.001 * np.arange(150) / 150.0, np.arange(150) / 150.0])[:, None]
    t, adj = tree_of(raw, 32)
    pairs = set(O.dense_pairs(t, adj))
    for a, b in pairs:
        assert (b, a) in pairs and t.box(a).is_leaf and t.box(b).is_leaf
    for b in t.boxes:
        if b.is_leaf:
            assert (b.id, b.id) in pairs
    assert adj.cross_level_adjacencies > 0


# ---------------------------------------------------------------- coloring
def chromatic(edges):
    n = len(edges)
    for k in range(1, n + 1):
        c = [-1] * n

        def go(v):
            if v == n:
                return True
            for col in range(k):
                if all(c[w] != col for w in edges[v] if w < v):
                    c[v] = col
                    if go(v + 1):
                        return True
            return False
        if go(0):
            return k


def test_dsatur_small_graphs():
    """proj/tests/test_coloring.cpp:91-113."""
    cyc = [sorted([(i + 1) % 5, (i - 1) % 5]) for i in range(5)]
    assert chromatic(cyc) == 3 and O.dsatur_color(cyc)[1] == 3
    k33 = [[3, 4, 5]] * 3 + [[0, 1, 2]] * 3
    assert chromatic(k33) == 2 and O.dsatur_color(k33)[1] == 2


def test_incompatibility_predicate():
    """proj/tests/test_coloring.cpp:128-149."""
    S = O.ConstraintSet
    assert O.incompatible(S(((10, 0),), (8, 9, 11), []), S(((8, 0),), (9, 10, 11), []))
    assert not O.incompatible(S(((1, 0),), (2,), []), S(((5, 0),), (6,), []))
    assert not O.incompatible(S(((3, 0),), (4,), []), S(((3, 0),), (5,), []))


def test_worked_example_colorings():
    """proj/tests/test_coloring.cpp:151-193."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    h1 = O.build_constraints(t, adj, 3, O.H1)
    assert sum(len(s.owners) for s in h1) == 18 and len(h1) == 12
    e = O.build_graph(h1)
    col, n = O.dsatur_color(e)
    assert n == 6 and all(col[v] != col[w] for v in range(len(e)) for w in e[v])
    l2 = O.build_constraints(t, adj, 2, O.H1)
    assert len(l2) == 4 and O.dsatur_color(O.build_graph(l2))[1] == 4
    u1 = O.build_constraints(t, adj, 3, O.UNIF1)
    assert len(u1) == 8 and O.dsatur_color(O.build_graph(u1))[1] == 5
    leaf = O.build_constraints(t, adj, 0, O.LEAF)
    assert O.dsatur_color(O.build_graph(leaf))[1] == 3
    assert all(len(s.zero) <= 2 for s in leaf)
    keys = [(s.payload, s.zero) for s in h1]
    assert len(set(keys)) == len(keys)


def test_constraints_satisfied_bit_exactly():
    """proj/tests/test_coloring.cpp:195-209 and payload reuse :228-248."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    for mode, width in [(O.H1, 12), (O.UNIF1, 12), (O.LEAF, t.max_leaf_size())]:
        level = 0 if mode == O.LEAF else 3
        sets = O.build_constraints(t, adj, level, mode)
        col, n = O.dsatur_color(O.build_graph(sets))
        mats = O.assemble_test_matrices(sets, col, n, t, 3, width, 77, 0)
        for i, s in enumerate(sets):
            omega = mats[col[i]].realize(t)
            for box, tag in s.payload:
                single = O.BlockTestMatrix(t.num_points, width, 77, 3, 0, [(box, tag)], [], [])
                pts = t.box(box).points
                assert np.array_equal(omega[pts], single.realize(t)[pts])
            for z in s.zero:
                assert not np.any(omega[t.box(z).points])
    sets = O.build_constraints(t, adj, 3, O.H1)
    col, n = O.dsatur_color(O.build_graph(sets))
    seen = {}
    for m in O.assemble_test_matrices(sets, col, n, t, 3, 10, 123, 0):
        om = m.realize(t)
        for box, _ in m.payload:
            rows = om[t.box(box).points]
            if box in seen:
                assert np.array_equal(seen[box], rows)
            seen[box] = rows


@pytest.mark.parametrize("d", [1, 2, 3])
def test_uniform_grid_color_bounds(d):
    """proj/tests/test_coloring.cpp:303-330."""
    per = 8 if d == 3 else 16
    t, adj = tree_of(O.uniform_grid_points(per, d), 1)
    assert t.is_fully_populated()
    for l in range(2, t.depth + 1):
        for mode, bound in [(O.H1, 6 ** d), (O.UNIF1, 5 ** d)]:
            sets = O.build_constraints(t, adj, l, mode)
            e = O.build_graph(sets)
            col, n = O.plan_coloring(t, sets, e, mode)
            assert n <= bound
            assert all(col[v] != col[w] for v in range(len(e)) for w in e[v])
    sets = O.build_constraints(t, adj, 0, O.LEAF)
    assert O.plan_coloring(t, sets, O.build_graph(sets), O.LEAF)[1] <= 3 ** d


# ---------------------------------------------------------------- linalg
def test_qr_and_pinv_properties():
    """proj/tests/test_linalg.cpp:43-113."""
    m = O.gaussian_matrix(50, 10, 3)
    q = O.qr_orthonormal(m)
    assert np.max(np.abs(q.T @ q - np.eye(10))) <= 1e-12
    deficient = m[:, :4] @ O.gaussian_matrix(4, 10, 4)
    assert O.qr_orthonormal(deficient).shape[1] == 4
    assert O.qr_orthonormal(m, 3).shape[1] == 3
    c = np.diag([3.0, 2.0, 1e-14])
    x = O.pinv_apply(c, np.eye(3))
    assert np.allclose(x, np.diag([1 / 3.0, 0.5, 0.0]))
    a = O.gaussian_matrix(8, 5, 5)
    b = O.gaussian_matrix(8, 2, 6)
    assert np.allclose(O.pinv_apply(a, b), np.linalg.lstsq(a, b, rcond=None)[0])
    assert not np.any(O.pinv_apply(np.zeros((4, 3)), np.ones((4, 2))))


# ---------------------------------------------------------------- driver
def dense_rel_error(truth, rep):
    got = rep.apply(np.eye(truth.shape[0]))
    return np.linalg.norm(truth - got, 2) / np.linalg.norm(truth, 2)


def test_exact_recovery_and_monotone_peeling():
    """proj/tests/test_peeling.cpp:28-53, :88-112."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    truth = O.synth_rank_structured(t, adj, 6, 77)
    rep, _ = O.compress(O.DenseOperator(truth), t, 6, 8, 20240601)
    assert dense_rel_error(truth, rep) <= 1e-9
    truth = O.synth_rank_structured(t, adj, 4, 11)
    rep, _ = O.compress(O.DenseOperator(truth), t, 4, 8, 20240601)
    for l in range(2, t.depth + 1):
        oracle = np.zeros_like(truth)
        for j in range(2, l + 1):
            for a, b in O.admissible_pairs(t, adj, j):
                oracle[np.ix_(t.box(a).points, t.box(b).points)] = truth[np.ix_(t.box(a).points, t.box(b).points)]
        got = rep.apply_truncated(l, np.eye(512))
        assert np.linalg.norm(oracle - got, 2) <= 1e-9 * np.linalg.norm(truth, 2)


def test_exact_recovery_adaptive_2d():
    """proj/tests/test_peeling.cpp:45-53."""
    t, adj = tree_of(O.random_cloud(700, 2, 31), 48)
    assert not t.is_fully_populated()
    truth = O.synth_rank_structured(t, adj, 5, 3)
    rep, _ = O.compress(O.DenseOperator(truth), t, 5, 8, 20240601)
    assert dense_rel_error(truth, rep) <= 1e-9


def test_sample_isolation():
    """proj/tests/test_peeling.cpp:55-86."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    truth = O.synth_rank_structured(t, adj, 4, 5)
    sets = O.build_constraints(t, adj, 2, O.H1)
    col, n = O.plan_coloring(t, sets, O.build_graph(sets), O.H1)
    mats = O.assemble_test_matrices(sets, col, n, t, 2, 10, 99, 0)
    for i, s in enumerate(sets):
        y = truth @ mats[col[i]].realize(t)
        for a, b in s.owners:
            rows, cols = t.box(a).points, t.box(b).points
            expect = truth[np.ix_(rows, cols)] @ O.payload_gaussian(t, b, 10, 99, 2, 0)
            assert np.max(np.abs(y[rows] - expect)) <= 1e-12 * np.max(np.abs(expect))


def test_leaf_diag_single_leaf_unit_capacity():
    """proj/tests/test_peeling.cpp:114-151."""
    t, adj = tree_of(O.equispaced_1d(256), 32)
    diag = np.diag(1.0 + 0.01 * np.arange(256))
    rep, _ = O.compress(O.DenseOperator(diag), t, 4, 8, 20240601)
    for (lam, mu), d in rep.dense.items():
        assert np.allclose(d, diag[np.ix_(t.box(lam).points, t.box(mu).points)], rtol=1e-12, atol=1e-12)
    t, adj = tree_of(O.equispaced_1d(48), 64)
    truth = O.gaussian_matrix(48, 48, 13)
    rep, _ = O.compress(O.DenseOperator(truth), t, 6, 8, 20240601)
    assert len(rep.dense) == 1 and np.max(np.abs(rep.dense[(0, 0)] - truth)) <= 1e-12
    t, adj = tree_of(O.equispaced_1d(32), 1)
    truth = O.synth_rank_structured(t, adj, 1, 5)
    rep, _ = O.compress(O.DenseOperator(truth), t, 1, 4, 20240601)
    assert dense_rel_error(truth, rep) <= 1e-9


def test_matvec_counts():
    """proj/tests/test_peeling.cpp:153-182."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    truth = O.synth_rank_structured(t, adj, 4, 21)
    r = 10
    _, rep1 = O.compress(O.DenseOperator(truth), t, 4, 6, 20240601)
    l3 = [p for p in rep1 if p["phase"] == "h1" and p["level"] == 3][0]
    assert (l3["colors"], l3["forward_cols"], l3["adjoint_cols"]) == (6, 6 * r, 6 * r)
    leaf = [p for p in rep1 if p["phase"] == "leaf"][0]
    assert (leaf["colors"], leaf["forward_cols"]) == (3, 3 * 64)
    t2, adj2 = tree_of(O.equispaced_1d(1024), 64)
    truth2 = O.synth_rank_structured(t2, adj2, 4, 21)
    _, rep2 = O.compress(O.DenseOperator(truth2), t2, 4, 6, 20240601)
    total = lambda rr: sum(p["forward_cols"] for p in rr)
    assert total(rep2) - total(rep1) == 6 * r


def test_dimension_mismatch_rejected():
    """proj/tests/test_peeling.cpp:347-352."""
    t, _ = tree_of(O.equispaced_1d(128), 32)
    with pytest.raises(ValueError):
        O.compress(O.DenseOperator(O.gaussian_matrix(64, 64, 3)), t, 6, 8, 1)


def test_power_method_on_exact_rep():
    """proj/tests/python/test_smoke.py:29-38 (err <= 1e-9 on exact inputs)."""
    t, adj = tree_of(O.equispaced_1d(512), 64)
    truth = O.synth_rank_structured(t, adj, 6, 11)
    op = O.DenseOperator(truth)
    rep, _ = O.compress(op, t, 6, 8, 3)
    assert O.rel_error_power_method(rep, op, 20, 5) <= 1e-9


def test_uniform_h1_driver_recovers_uniform_synthetic():
    """acceptance.cpp:75-93 for PeelFormat::kUnifH1 (criterion 1's recovery
    check): the uniform driver of the oracle (SVD bases, peeling.cpp:292-454)
    recovers a uniform rank-structured synthetic to 1e-9 in 1D and 2D, with
    fewer matvec columns than the H1 driver on the same tree."""
    for pts, leaf in ((O.equispaced_1d(512), 64), (O.random_cloud(600, 2, 5), 48)):
        t, adj = tree_of(pts, leaf)
        truth = O.synth_rank_structured(t, adj, 6, 11, fmt="unif-h1")
        rep, report = O.compress(O.DenseOperator(truth), t, 6, 8, O.mix_seed(11, 1), fmt="unif-h1")
        got = rep.apply(np.eye(t.num_points))
        assert np.linalg.norm(got - truth, 2) <= 1e-9 * np.linalg.norm(truth, 2)
        _, report_h1 = O.compress(O.DenseOperator(truth), t, 6, 8, O.mix_seed(11, 1))
        cols = lambda rp: sum(p["forward_cols"] + p["adjoint_cols"] for p in rp)
        assert cols(report) < cols(report_h1)
