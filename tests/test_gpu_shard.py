"""Sharded compression on one GPU by emulation: splitting the K2 / K6
launches and the per-pair K4 QR / K5 B-solve batches into the per-rank work
ranges (as N ranks would before their NCCL broadcasts of samples, factors and
ranks) reproduces the single-rank samples, factors and dense blocks bit for
bit (each tile and each pair is computed by exactly one rank)."""
import numpy as np
import pytest

from paper_2205_03406_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,shards", [("c3", 16384, 2), ("c3", 16384, 3), ("c3", 16384, 8),
                                           ("c4", 16384, 3)])
def test_emulated_shards_bit_identical(hp, gpu_available, name, n, shards):
    w = configs.scaled(name, n)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    one = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True)
    many = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True,
                       emulate_shards=shards)
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            assert np.array_equal(one.captured(l, i), many.captured(l, i))
            for a, b in zip(one.block(l, i), many.block(l, i)):
                assert np.array_equal(a, b)
    for i in range(len(t.dense_pairs())):
        assert np.array_equal(one.dense_block(i), many.dense_block(i))


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
