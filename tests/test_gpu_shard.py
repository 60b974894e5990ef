"""Owner-computes sharded compression on one GPU: `world`
ranks emulated by threads (hp_compress_group: the same sharded driver, device
copies in place of NCCL). Every pair's samples, U, V, B and every dense block
equal the single-rank run bit for bit on the rank(s) that hold them, every
block is held by its owners, and each rank's arena is about 1/world of the
whole (plus the cut-crossing pairs held by both owners)."""
import numpy as np
import pytest

from paper_2205_03406_b200 import configs

pytestmark = pytest.mark.gpu


def _check_group(hp, t, one, many, world):
    owner, cut, _ = hp.shard_owners(t, world)
    for l in range(2, t.depth + 1):
        pairs = t.admissible_pairs(l)
        for i, (a, b) in enumerate(pairs):
            holders = [g for g in range(world) if many[g].holds(l, i)]
            if l < cut:
                assert holders == list(range(world)), (l, i)
            else:
                assert set(holders) == {int(owner[a]), int(owner[b])}, (l, i, holders)
                ref = one.captured(l, i)
                got = many[int(owner[a])].captured(l, i)
                assert np.array_equal(ref, got), ("samples", l, i)
            want = one.block(l, i)
            for g in holders:
                for x, y in zip(want, many[g].block(l, i)):
                    assert np.array_equal(x, y), ("factors", l, i, g)
    for i, (lam, mu) in enumerate(t.dense_pairs()):
        holders = [g for g in range(world) if many[g].holds(-1, i)]
        assert holders == [int(owner[lam])]
        assert np.array_equal(one.dense_block(i), many[holders[0]].dense_block(i))


@pytest.mark.parametrize("name,n,world", [("c3", 16384, 2), ("c3", 16384, 3), ("c3", 16384, 8),
                                          ("c4", 16384, 3), ("c2", 8192, 4), ("c1", 4096, 2)])
def test_sharded_group_bit_identical(hp, gpu_available, name, n, world):
    w = configs.scaled(name, n)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    one = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    many = hp.compress_group(op, t, world, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    assert [m.shard() for m in many] == [(world, g) for g in range(world)]
    _check_group(hp, t, one, many, world)
    f_one, d_one = one.sizes()
    sizes = [m.sizes() for m in many]
    assert sum(s[1] for s in sizes) == d_one
    for g, (f, d) in enumerate(sizes):
        assert (f, d) == hp.export_sizes(t, w.rank, world, g)
    # each pair is counted once over the group
    assert sum(m.storage()["total"] for m in many) == one.storage()["total"]


def test_sharded_c4_arena_fraction(hp, gpu_available):
    """Config 4 (sphere, octree) at N = 2^17 on 8 emulated ranks: bit-identical
    to one rank, and no rank holds more than 1/8 of the factors plus its
    cut-crossing duplicates (bounded here at 1.6 / 8)."""
    w = configs.scaled("c4", 131072)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    world = 8
    one = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    many = hp.compress_group(op, t, world, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    _check_group(hp, t, one, many, world)
    f_one, d_one = one.sizes()
    for m in many:
        f, d = m.sizes()
        assert f <= 1.6 * f_one / world
        assert m.report["peak_device_bytes"] > 0
    peaks = [m.report["peak_device_bytes"] for m in many]
    print("per-rank peak device bytes", peaks, "single", one.report["peak_device_bytes"])


@pytest.mark.parametrize("name,n", [("c3", 32768), ("c5", 16384)])
def test_level_overlap_bit_identical(hp, gpu_available, name, n, monkeypatch):
    """Level l+1's K1/K2 run on the apply stream while level l peels, factors
    and solves on the main stream (driver.cu ApplyStage); the overlapped run
    and the serialized one (HP_SERIAL_LEVELS=1) give identical factors and
    dense blocks (no capture: capture synchronizes inside each level).
    HP_SERIAL_LEVELS=0 forces the overlap where the driver would not choose
    it (FP64 DMMA K2, config 5)."""
    w = configs.scaled(name, n)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    monkeypatch.setenv("HP_SERIAL_LEVELS", "0")
    over = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    monkeypatch.setenv("HP_SERIAL_LEVELS", "1")
    ser = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            for a, b in zip(over.block(l, i), ser.block(l, i)):
                assert np.array_equal(a, b)
    for i in range(len(t.dense_pairs())):
        assert np.array_equal(over.dense_block(i), ser.dense_block(i))
