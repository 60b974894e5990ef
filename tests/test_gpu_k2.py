"""K2 variants agree bit for bit: the checked evaluation path (i == j and
coincident-point tests, forced by k2 mode bit 3) and the fused kernel (mode bit
2) reproduce the default warp-specialized, unchecked samples exactly (same
kernel values, same DMMA accumulation order per output element)."""
import numpy as np
import pytest

from paper_2205_03406_b200 import _lib, configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c2", "c3"])
@pytest.mark.parametrize("mode", [8, 4])
def test_k2_variants_bit_identical(hp, gpu_available, name, mode):
    w = configs.scaled(name, 8192)
    pts = w.points()
    t = hp.build_tree(pts, w.leaf)
    op = hp.kernel_operator(w.kernel, pts, w.param)
    reps = []
    hp.set_k2_path("fp64")  # the FP64 DMMA kernels (the int8 path: test_gpu_k2_int8.py)
    try:
        for m in (0, mode):
            _lib.lib().hp_debug_set_k2_mode(m)
            reps.append(hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7, capture=True))
    finally:
        _lib.lib().hp_debug_set_k2_mode(0)
        hp.set_k2_path("int8")
    for l in range(2, t.depth + 1):
        for i in range(len(t.admissible_pairs(l))):
            assert np.array_equal(reps[0].captured(l, i), reps[1].captured(l, i))
