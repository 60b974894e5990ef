"""The .hrep file format (proj/src/serialize.cpp): the oracle's writer and
reader round-trip an oracle H1 representation byte for byte, the dense
matrix file layout matches, and (GPU) the device writer produces exactly the
oracle writer's bytes for the same blocks, the device reader loads an
oracle-written file whose apply matches the oracle's, and save -> load ->
save is byte-identical (the reference's round-trip test,
proj/tests/test_hmatrix.cpp:204-233)."""
import os
import struct

import numpy as np
import pytest

import oracle as O


def _oracle_rep(n=512, leaf=32, k=5):
    pts = O.equispaced_1d(n)
    tree = O.BoxTree(O.PointCloud(pts), leaf)
    truth = O.synth_rank_structured(tree, O.adjacency(tree), k, 3)
    rep, _ = O.compress(O.DenseOperator(truth), tree, k, 4, 11)
    return pts, tree, truth, rep


def test_oracle_hrep_round_trip():
    _, tree, _, rep = _oracle_rep()
    data = O.save_rep_bytes(rep, 5, 32)
    meta, boxes, levels, dense = O.load_rep_bytes(data)
    assert meta["format"] == 1 and meta["n"] == tree.num_points and meta["rank"] == 5
    assert meta["depth"] == tree.depth and meta["dense_ready"]
    assert len(boxes) == len(tree.boxes)
    for (lvl, parent, coord, children, points), b in zip(boxes, tree.boxes):
        assert (lvl, parent, tuple(coord), list(children), list(points)) == (
            b.level, b.parent, tuple(b.coord), list(b.children), [int(p) for p in b.points])
    for l, lv in enumerate(levels):
        assert set(lv) == set(rep.levels[l])
        for key, (u, bb, v) in lv.items():
            for x, y in zip((u, bb, v), rep.levels[l][key]):
                assert np.array_equal(x, y)
    assert set(dense) == set(rep.dense)
    # magic and meta layout (serialize.cpp:155-158, :128-138)
    assert struct.unpack_from("<Q", data, 0)[0] == 0x3150524C45455048
    assert data[8] == 1


def test_dense_matrix_file_layout():
    m = np.arange(6.0).reshape(2, 3)
    data = O.save_dense_matrix_bytes(m)
    assert struct.unpack_from("<Qqq", data, 0) == (0x314D444C45455048, 2, 3)
    assert np.array_equal(np.frombuffer(data, "<f8", offset=24).reshape(2, 3, order="F"), m)


def test_dense_matrix_file_round_trip(hp, tmp_path):
    """save_dense_matrix / load_dense_matrix (host code, no GPU needed)."""
    m = np.random.default_rng(77).standard_normal((20, 30))
    path = str(tmp_path / "dense_test.bin")
    hp.save_dense_matrix(path, m)
    assert open(path, "rb").read() == O.save_dense_matrix_bytes(m)
    assert np.array_equal(hp.load_dense_matrix(path), m)


@pytest.mark.gpu
def test_device_hrep_matches_oracle_writer(hp, gpu_available, tmp_path):
    pts = O.random_cloud(3000, 2, O.mix_seed(7, 0xF2))
    tree = hp.build_tree(pts, 64)
    op = hp.kernel_operator("log", pts, 1.0)
    rep = hp.compress(op, tree, rank=10, oversample=6, seed=7)
    path = str(tmp_path / "dev.hrep")
    rep.save(path)
    data = open(path, "rb").read()
    meta, boxes, levels, dense = O.load_rep_bytes(data)
    assert meta["rank"] == 10 and meta["built_level"] == tree.depth and meta["dense_ready"]
    # every block equals the device's block() read-back, bit for bit
    for l in range(2, tree.depth + 1):
        pairs = tree.admissible_pairs(l)
        assert sorted(levels[l]) == sorted(pairs)
        for i, key in enumerate(pairs):
            for x, y in zip(levels[l][key], rep.block(l, i)):
                assert np.array_equal(x, y)
    for i, key in enumerate(tree.dense_pairs()):
        assert np.array_equal(dense[key], rep.dense_block(i))
    # load -> save reproduces the bytes; the loaded rep applies identically
    back = hp.load_rep(path)
    path2 = str(tmp_path / "dev2.hrep")
    back.save(path2)
    assert open(path2, "rb").read() == data
    x = np.random.default_rng(8).standard_normal((3000, 3))
    assert np.array_equal(back.apply(x), rep.apply(x))


@pytest.mark.gpu
def test_device_loads_oracle_hrep(hp, gpu_available, tmp_path):
    pts, tree, truth, rep = _oracle_rep()
    path = str(tmp_path / "oracle.hrep")
    open(path, "wb").write(O.save_rep_bytes(rep, 5, 32))
    back = hp.load_rep(path)
    x = np.random.default_rng(9).standard_normal((tree.num_points, 2))
    want = rep.apply(x) if hasattr(rep, "apply") else None
    got = back.apply(x)
    if want is not None:
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    path2 = str(tmp_path / "again.hrep")
    back.save(path2)
    assert open(path2, "rb").read() == open(path, "rb").read()
