"""Bit-exact parity of the product's host planning layer (C++ behind the C
ABI) with the oracle: trees, adjacency, admissible/dense pairs, constraint
sets, incompatibility graphs, DSatur/tile colorings and per-color payload
lists. Runs without a GPU."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2205_03406_b200 import configs


ROOT_DIR = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def geometries():
    yield "worked-1d", O.equispaced_1d(512), 64
    yield "figure", O.equispaced_1d(400), 100
    yield "random-2d", O.random_cloud(700, 2, 31), 48
    yield "random-2d-b", O.random_cloud(1000, 2, 99), 50
    yield "lopsided", np.concatenate([0.001 * np.arange(150) / 150.0, np.arange(150) / 150.0])[:, None], 32
    yield "grid-2d", O.uniform_grid_points(16, 2), 1
    yield "grid-3d", O.uniform_grid_points(8, 3), 1
    yield "c1", configs.make_points("c1", 4096), 64
    yield "c2-scaled", configs.make_points("c2", 8192), 64
    yield "c3-scaled", configs.make_points("c3", 8192), 128
    yield "c4-scaled", configs.make_points("c4", 16384), 256
    yield "c5-scaled", configs.make_points("c5", 8192), 256


GEOMS = list(geometries())


@pytest.mark.parametrize("name,pts,leaf", GEOMS, ids=[g[0] for g in GEOMS])
def test_tree_and_adjacency_bit_exact(hp, name, pts, leaf):
    t = hp.build_tree(pts, leaf)
    ot = O.BoxTree(O.PointCloud(pts), leaf)
    oadj = O.adjacency(ot)
    _trees_equal(t, ot, oadj)


def _trees_equal(t, ot, oadj):
    assert (t.depth, t.num_boxes, t.num_points) == (ot.depth, ot.num_boxes, ot.num_points)
    assert t.fully_populated == ot.is_fully_populated()
    assert t.max_leaf_size == ot.max_leaf_size()
    for b in ot.boxes:
        assert t.box_level(b.id) == b.level
        assert t.box_parent(b.id) == b.parent
        assert tuple(t.box_coord(b.id)) == b.coord
        assert t.box_points(b.id) == [int(p) for p in b.points]
        assert t.children(b.id) == b.children
        assert t.neighbors(b.id) == oadj.neighbors[b.id]
        assert t.interaction(b.id) == oadj.interaction[b.id]
        assert t.coarse_leaf_neighbors(b.id) == oadj.coarse_leaf_neighbors[b.id]
        assert t.dense_partners(b.id) == oadj.dense_partners[b.id]
    assert t.cross_level_adjacencies == oadj.cross_level_adjacencies
    for l in range(2, ot.depth + 1):
        assert t.admissible_pairs(l) == O.admissible_pairs(ot, oadj, l)
    assert t.dense_pairs() == O.dense_pairs(ot, oadj)


def _compare_plan(hp, t, ot, oadj, level, mode, omode):
    p = hp.plan(t, level, mode, 12, 7, 0)
    sets = O.build_constraints(ot, oadj, level, omode)
    assert p.n_vertices == len(sets)
    for got, want in zip(p.sets, sets):
        assert tuple(tuple(x) for x in got["payload"]) == want.payload
        assert tuple(got["zero"]) == want.zero
        assert [tuple(o) for o in got["owners"]] == want.owners
    if len(sets) <= 2500:  # the oracle's three graph builds agree with the literal O(V^2) scan
        from oracle import hpeel_ref
        lit = O.build_graph_literal(sets)
        assert lit == O.build_graph(sets) == hpeel_ref._build_graph_indexed(sets)
    if True:
        edges = O.build_graph(sets)
        assert p.edges == edges
        col, n = O.plan_coloring(ot, sets, edges, omode)
        assert p.color == col and p.n_colors == n
        dcol, dn = O.dsatur_color(edges)
        assert p.dsatur_color == dcol and p.dsatur_colors == dn
        basis = {b.id: np.zeros((0, 12)) for b in ot.boxes} if omode == O.UNIF2 else None
        mats = O.assemble_test_matrices(sets, col, n, ot, level, 12, 7, 0, basis)
        assert p.color_payload == [[b for b, _ in m.payload] for m in mats]
    return p


@pytest.mark.parametrize("name,pts,leaf", GEOMS, ids=[g[0] for g in GEOMS])
def test_level_and_leaf_plans_bit_exact(hp, name, pts, leaf):
    t = hp.build_tree(pts, leaf)
    ot = O.BoxTree(O.PointCloud(pts), leaf)
    oadj = O.adjacency(ot)
    for l in range(2, ot.depth + 1):
        _compare_plan(hp, t, ot, oadj, l, "h1", O.H1)
        _compare_plan(hp, t, ot, oadj, l, "unif-stage1", O.UNIF1)
        _compare_plan(hp, t, ot, oadj, l, "unif-stage2", O.UNIF2)
    _compare_plan(hp, t, ot, oadj, ot.depth, "leaf", O.LEAF)


def _plans_equal_at_scale(hp, t, ot, oadj, levels, leaf=True):
    """Constraint sets, DSatur / plan colorings and per-color payload lists of
    the product (implicit graph, the path compress() takes) equal the
    oracle's (indexed graph build, same edge set as the pairwise scan)."""
    modes = [("h1", O.H1, l) for l in levels] + ([("leaf", O.LEAF, ot.depth)] if leaf else [])
    for mode, omode, level in modes:
        p = hp.plan(t, level, mode, 12, 7, 0, implicit=True)
        op = O.make_plan(ot, oadj, level, omode, 12, 7, 0)
        assert p.n_vertices == len(op.sets), (mode, level)
        if not op.sets:
            continue
        for got, want in zip(p.sets, op.sets):
            assert tuple(got["zero"]) == want.zero and got["payload"][0][0] == want.payload[0][0]
        assert p.color == list(op.color), (mode, level)
        assert p.n_colors == len(op.matrices)
        assert p.color_payload == [[b for b, _ in m.payload] for m in op.matrices], (mode, level)


def test_full_size_c3_planning_bit_exact(hp):
    """Config 3 at its full N = 2^18 (the bench workload): tree, adjacency,
    pair lists and every H1 level's and the leaf phase's coloring equal the
    oracle's."""
    pts = configs.make_points("c3", 262144)
    t = hp.build_tree(pts, 128)
    ot = O.BoxTree(O.PointCloud(pts), 128)
    oadj = O.adjacency(ot)
    _trees_equal(t, ot, oadj)
    _plans_equal_at_scale(hp, t, ot, oadj, range(2, ot.depth + 1))


@pytest.mark.gpu  # CPU-only but ~10 minutes of oracle planning: runs with the GPU-box suite
@pytest.mark.timeout(3600)
def test_full_size_c4_planning_bit_exact(hp):
    """Config 4 at N = 2^20 (the north-star target): tree, adjacency, pair
    lists and every H1 level's coloring equal the oracle's. (Its leaf
    graph, 1.5e9 edges, is beyond the oracle's reach.)"""
    pts = configs.make_points("c4", 1 << 20)
    t = hp.build_tree(pts, 256)
    ot = O.BoxTree(O.PointCloud(pts), 256)
    oadj = O.adjacency(ot)
    _trees_equal(t, ot, oadj)
    _plans_equal_at_scale(hp, t, ot, oadj, range(2, ot.depth + 1), leaf=False)


def test_inverted_index_graph_equals_pairwise_scan(hp):
    """build_graph's inverted index gives the literal scan's edge set
    (proj/src/coloring.cpp:154-167) on every level of an adaptive tree."""
    pts = configs.make_points("c3", 16384)
    t = hp.build_tree(pts, 128)
    for l in range(2, t.depth + 1):
        fast = hp.plan(t, l, "h1", 8, 1, 0)
        slow = hp.plan(t, l, "h1", 8, 1, 0, pairwise=True)
        assert fast.edges == slow.edges and fast.color == slow.color
    fast = hp.plan(t, t.depth, "leaf", 8, 1, 0)
    slow = hp.plan(t, t.depth, "leaf", 8, 1, 0, pairwise=True)
    assert fast.edges == slow.edges and fast.color == slow.color


def test_worked_example_known_answers(hp):
    """proj/tests/test_coloring.cpp:151-182, proj/tests/python/test_smoke.py:14-26."""
    t = hp.build_tree(hp.equispaced_1d(512), 64)
    assert t.depth == 3 and t.num_points == 512
    assert len(t.admissible_pairs(3)) == 18 and len(t.admissible_pairs(2)) == 6
    h1 = hp.level_coloring(t, 3, "h1")
    assert h1["n_vertices"] == 12 and h1["n_colors"] == 6
    assert hp.level_coloring(t, 2, "h1")["n_colors"] == 4
    assert hp.level_coloring(t, 3, "unif-stage1") == {"n_vertices": 8, "n_edges": 22, "n_colors": 5}
    assert hp.level_coloring(t, 3, "leaf")["n_colors"] == 3


def test_dsatur_known_answers(hp):
    """proj/tests/test_coloring.cpp:91-126."""
    cyc = [sorted([(i + 1) % 5, (i - 1) % 5]) for i in range(5)]
    assert hp.dsatur(cyc)["num_colors"] == 3
    k33 = [[3, 4, 5]] * 3 + [[0, 1, 2]] * 3
    assert hp.dsatur(k33)["num_colors"] == 2
    t = hp.build_tree(hp.equispaced_1d(4096), 32)
    p = hp.plan(t, t.depth, "h1", 4, 0, 0)
    v = p.n_vertices
    deg = max(len(e) for e in p.edges)
    assert p.queue_ops <= 4.0 * (deg + 1.0) * v * max(1.0, np.log2(v))


def test_gaussian_stream_and_realize_bit_exact(hp):
    """Host RNG equals the frozen stream (libm path, bit for bit), and
    BlockTestMatrix::realize matches the oracle on every color."""
    for rows, cols, seed in [(4, 3, 7), (17, 13, 2**62 + 3), (1, 1, 0)]:
        assert np.array_equal(hp.gaussian_matrix(rows, cols, seed), O.gaussian_matrix_libm(rows, cols, seed))
    assert np.array_equal(hp.random_cloud(9, 3, 11), O.random_cloud(9, 3, 11))
    assert hp.mix_seed(7, 0xC1) == O.mix_seed(7, 0xC1)
    t = hp.build_tree(hp.equispaced_1d(512), 64)
    ot = O.BoxTree(O.PointCloud(O.equispaced_1d(512)), 64)
    oadj = O.adjacency(ot)
    for mode, omode, level in [("h1", O.H1, 3), ("leaf", O.LEAF, 3)]:
        width = 12 if mode == "h1" else 64
        p = hp.plan(t, level, mode, width, 77, 1)
        sets = O.build_constraints(ot, oadj, level, omode)
        col, n = O.plan_coloring(ot, sets, O.build_graph(sets), omode)
        mats = O.assemble_test_matrices(sets, col, n, ot, level, width, 77, 1)
        for c in range(n):
            got = p.realize(c)
            want = mats[c].realize(ot)
            assert np.max(np.abs(got - want)) <= 4e-16 * max(1.0, np.max(np.abs(want)))


def test_error_behaviour(hp):
    """Exception mapping of the C ABI: invalid_argument -> ValueError,
    runtime_error -> RuntimeError (proj/src/box_tree.cpp:130-133)."""
    with pytest.raises(RuntimeError):
        hp.build_tree(np.zeros((10, 1)), 2)
    with pytest.raises(ValueError):
        hp.build_tree(np.zeros((0, 1)), 2)
    with pytest.raises(ValueError):
        hp.build_tree(np.array([[0.0], [np.nan]]), 2)
    with pytest.raises(ValueError):
        hp.build_tree(hp.equispaced_1d(16), 0)


def test_export_sizes_match_layout(hp):
    """hp_export_sizes: U, V, B per admissible pair of every level plus the
    compact |I_lam| x |I_mu| dense blocks (D = Y(I_lam, 0:|I_mu|),
    proj/src/peeling.cpp:513-517; H1Rep::export_all layout)."""
    pts = O.random_cloud(3000, 2, O.mix_seed(7, 0xE3))
    tree = hp.build_tree(pts, 32)
    ot = O.BoxTree(O.PointCloud(pts), 32)
    k = 9
    want_f = 0
    for level in range(2, tree.depth + 1):
        for a, b in tree.admissible_pairs(level):
            want_f += (len(ot.box(a).points) + len(ot.box(b).points)) * k + k * k
    want_d = sum(len(ot.box(lam).points) * len(ot.box(mu).points) for lam, mu in tree.dense_pairs())
    assert hp.export_sizes(tree, k) == (want_f, want_d)
    # sharded layouts: every dense block on exactly one rank, every pair on its
    # owners (both for a cut-crossing pair), replicated levels on every rank
    for world in (2, 3, 8):
        owner, cut, bounds = hp.shard_owners(tree, world)
        assert bounds[0] == 0 and bounds[-1] == tree.num_points and all(np.diff(bounds) >= 0)
        f_tot = d_tot = 0
        for g in range(world):
            f, d = hp.export_sizes(tree, k, world, g)
            f_tot += f
            d_tot += d
        assert d_tot == want_d
        want_fw = 0
        for level in range(2, tree.depth + 1):
            for a, b in tree.admissible_pairs(level):
                size = (len(ot.box(a).points) + len(ot.box(b).points)) * k + k * k
                if level < cut:
                    want_fw += world * size
                else:
                    assert owner[a] >= 0 and owner[b] >= 0
                    want_fw += size * (1 if owner[a] == owner[b] else 2)
        assert f_tot == want_fw


def test_shard_ownership_is_a_contiguous_partition(hp):
    """Boxes at or below the cut belong to exactly one rank, a box's rank owns
    its whole tree-order range, and the ranks' point counts are balanced at
    frontier-box granularity."""
    w = configs.scaled("c3", 16384)
    t = hp.build_tree(w.points(), w.leaf)
    lvl, parent, _, off, _ = t._box_arrays()
    for world in (2, 4, 8):
        owner, cut, bounds = hp.shard_owners(t, world)
        for b in range(t.num_boxes):
            if lvl[b] >= cut or not t.children(b):
                assert 0 <= owner[b] < world
            else:
                assert owner[b] == -1
            if parent[b] >= 0 and owner[parent[b]] >= 0:
                assert owner[b] == owner[parent[b]]
        counts = np.diff(bounds)
        assert counts.sum() == t.num_points and counts.min() > 0


@pytest.mark.parametrize("name,pts,leaf", GEOMS, ids=[g[0] for g in GEOMS])
def test_implicit_graph_dsatur_equals_explicit(hp, name, pts, leaf):
    """compress() colors single-payload constraint sets (H1 and leaf modes)
    without materializing the graph; its DSatur coloring, color count and
    plan coloring equal the explicit graph's."""
    t = hp.build_tree(pts, leaf)
    modes = [("leaf", t.depth)] + [("h1", l) for l in range(2, t.depth + 1)]
    for mode, level in modes:
        a = hp.plan(t, level, mode, 8, 7, 0)
        b = hp.plan(t, level, mode, 8, 7, 0, implicit=True)
        if a.n_vertices == 0:
            continue
        assert a.dsatur_color == b.dsatur_color, (name, mode, level)
        assert a.dsatur_colors == b.dsatur_colors and a.n_colors == b.n_colors
        assert a.color == b.color and a.color_payload == b.color_payload, (name, mode, level)


def test_threaded_dsatur_equals_serial():
    """The tournament-tree DSatur with threaded neighbor sweeps (used for the
    big leaf graphs, e.g. 1.5e9 edges at config 4) colors exactly like the
    serial heap implementation and the explicit graph: forced on with every
    sweep threaded (HP_DSATUR_SWEEP_MIN=0), in a fresh process."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_2205_03406_b200 as hp\n"
        "from paper_2205_03406_b200 import configs\n"
        "for name, n, leaf in [('c3', 16384, 128), ('c4', 16384, 256), ('c5', 8192, 256), ('c2', 8192, 64)]:\n"
        "    t = hp.build_tree(configs.make_points(name, n), leaf)\n"
        "    for mode, level in [('leaf', t.depth)] + [('h1', l) for l in range(2, t.depth + 1)]:\n"
        "        a = hp.plan(t, level, mode, 8, 7, 0)\n"
        "        b = hp.plan(t, level, mode, 8, 7, 0, implicit=True)\n"
        "        assert a.dsatur_color == b.dsatur_color and a.color == b.color, (name, mode, level)\n"
        "print('ok')\n" % ROOT_DIR)
    env = dict(os.environ, HP_DSATUR_THREADS="4", HP_DSATUR_SWEEP_MIN="0")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("d,per", [(1, 32), (2, 16), (3, 8)])
def test_fallback_pattern_plans_match_oracle(hp, d, per):
    """ColoringStrategy::kFallbackPattern (proj/src/coloring.cpp:334-407,
    proj/src/peeling.cpp:131-153): per pattern matrix the payload boxes, and
    the block -> matrix map, for the H1 pairs of every level, the uniform
    stage-1 boxes and the leaf probes; dense realizations agree (same nonzero
    pattern, values to the last bits of the numpy vs libm Box-Muller)."""
    pts = O.uniform_grid_points(per, d)
    t = hp.build_tree(pts, 1)
    ot = O.BoxTree(O.PointCloud(pts), 1)
    oadj = O.adjacency(ot)
    assert t.fully_populated
    for mode, omode, levels in (("h1", O.H1, range(2, t.depth + 1)), ("unif-stage1", O.UNIF1, range(2, t.depth + 1)),
                                ("leaf", O.LEAF, [t.depth])):
        for l in levels:
            got = hp.Plan(t, l, mode, 3, 7, 0, strategy="fallback-pattern")
            want = O.make_plan(ot, oadj, l, omode, 3, 7, 0, strategy="fallback-pattern")
            assert got.n_colors == len(want.matrices) == {"h1": 6, "unif-stage1": 5, "leaf": 3}[mode] ** d
            assert got.color_payload == [[b for b, _ in m.payload] for m in want.matrices]
            wmap = dict(want.block_to_matrix)
            wmap.update({(a, -1): c for a, c in want.box_to_matrix.items()})
            assert got.block_to_matrix() == wmap
            for c in (0, got.n_colors // 2, got.n_colors - 1):
                a, b = got.realize(c), want.matrices[c].realize(ot)
                assert np.array_equal(a != 0, b != 0)
                assert np.max(np.abs(a - b)) <= 4e-16 * max(1.0, np.max(np.abs(b)))  # numpy vs libm log / sincos


def test_fallback_pattern_needs_a_full_tree(hp):
    t = hp.build_tree(O.random_cloud(300, 2, 3), 16)
    assert not t.fully_populated
    with pytest.raises(ValueError):
        hp.Plan(t, 2, "h1", 3, 7, 0, strategy="fallback-pattern")
