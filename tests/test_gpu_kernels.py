"""Kernel-level parity probes of the sm_100a path through the C ABI."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_log_accuracy(hp, gpu_available):
    """The log-kernel black box evaluates log on the device with its own
    argument reduction (device.cuh fast_log); <= 2 ulp against libm."""
    rng = np.random.default_rng(0)
    x = np.concatenate([
        np.exp(rng.uniform(-700, 700, 200000)),
        1.0 + rng.uniform(-1e-3, 1e-3, 50000),
        rng.uniform(0.5, 2.0, 50000),
        np.array([1.0, 2.0, 0.5, math.sqrt(2.0), math.sqrt(0.5), 1e-300, 1e300, 3.0]),
    ])
    got = hp.debug_log(x)
    want = np.array([math.log(v) for v in x])
    ulp = np.spacing(np.abs(want))
    err = np.abs(got - want)
    # absolute bound near x = 1 (log -> 0), 2 ulp elsewhere
    assert np.all(err <= np.maximum(2.0 * ulp, 2.2e-16 * np.abs(x - 1.0) + 1e-300))
