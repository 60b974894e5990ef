"""Streamed export (hp_compress_export): the host arrays filled while the
representation is built equal a bulk export after compress, bit for bit,
for pinned (asynchronous, per level) and pageable (deferred) destinations."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pinned", [True, False])
def test_streamed_export_equals_bulk(hp, gpu_available, pinned):
    pts = O.random_cloud(6000, 2, O.mix_seed(7, 0xE1))
    tree = hp.build_tree(pts, 64)
    op = hp.kernel_operator("log", pts, 1.0)
    nf, nd = hp.export_sizes(tree, 12)
    rep = hp.compress(op, tree, rank=12, oversample=6, seed=7)
    assert rep.sizes() == (nf, nd)
    want_f, want_d = np.empty(nf), np.empty(nd)
    rep.export(want_f, want_d)
    alloc = hp.pinned_empty if pinned else np.empty
    hf, hd = alloc(nf), alloc(nd)
    hf[:] = np.nan
    hd[:] = np.nan
    rep2 = hp.compress(op, tree, rank=12, oversample=6, seed=7, export_to=(hf, hd))
    assert np.array_equal(hf, want_f)
    assert np.array_equal(hd, want_d)
    # the streamed rep is a normal representation too
    x = np.random.default_rng(0).standard_normal((6000, 2))
    assert np.array_equal(rep2.apply(x), rep.apply(x))


def test_export_arrays_too_small(hp, gpu_available):
    pts = O.random_cloud(2000, 1, O.mix_seed(7, 0xE2))
    tree = hp.build_tree(pts, 64)
    op = hp.kernel_operator("log", pts, 1.0)
    nf, nd = hp.export_sizes(tree, 8)
    with pytest.raises(ValueError):
        hp.compress(op, tree, rank=8, oversample=4, export_to=(np.empty(nf - 1), np.empty(nd)))
