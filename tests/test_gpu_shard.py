"""Sharded black-box apply on one GPU by emulation: splitting the K2 / K6
launches into the per-rank work ranges (as N ranks would before their NCCL
broadcast) reproduces the single-rank samples, factors and dense blocks bit
for bit (each tile is computed by exactly one rank)."""
import numpy as np
import pytest

from paper_2205_03406_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_emulated_shards_bit_identical(hp, gpu_available, shards):
    w = configs.scaled("c3", 16384)
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
