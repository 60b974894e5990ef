"""Synthetic BASELINE.json workloads, master seed S0 = 7.

BASELINE.json names no public dataset; these seeded generators reproduce the
shapes, sizes and point distributions of its five configs. Geometry streams
use the reference's own generators (random_cloud, gaussian_matrix:
proj/src/operators.cpp:88-95, proj/src/rng.cpp:35-59) through the C ABI.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

S0 = 7


def _gen(gen):
    """The point generators (random_cloud, gaussian_matrix, mix_seed): the
    package's C ABI by default; bench.py's reference arm passes the oracle's
    restatement so that arm never loads the product library."""
    if gen is None:
        import paper_2205_03406_b200 as pkg  # the C ABI loads on first call
        return pkg
    return gen


@dataclass
class Workload:
    name: str
    n: int
    dim: int
    kernel: str          # "log" | "invdist4pi" | "exp"
    dense: bool          # explicit dense A as the black box (config 1)
    leaf: int
    rank: int
    oversample: int
    param: float = 1.0
    description: str = ""

    def points(self, gen=None) -> np.ndarray:
        return make_points(self.name, self.n, gen)


def starfish_points(n: int, seed: int, gen=None) -> np.ndarray:
    """Config 3: r(t) = 1 + 0.3 cos 5t; half the parameters uniform on
    [0, 2 pi), half on [0, t*) where t* is the first grid point t_j = 2 pi j / 2^20
    whose trapezoid-rule arclength reaches 10% of the total."""
    u = _gen(gen).random_cloud(n, 1, seed)[:, 0]
    m = 1 << 20
    t = 2.0 * math.pi * np.arange(m + 1) / m
    r = 1.0 + 0.3 * np.cos(5.0 * t)
    rp = -1.5 * np.sin(5.0 * t)
    speed = np.sqrt(r * r + rp * rp)
    s = np.concatenate([[0.0], np.cumsum(0.5 * (speed[1:] + speed[:-1]) * (t[1] - t[0]))])
    j = int(np.searchsorted(s, 0.1 * s[-1], side="left"))
    tstar = t[j]
    half = n // 2
    tt = np.empty(n)
    tt[:half] = 2.0 * math.pi * u[:half]
    tt[half:] = tstar * u[half:]
    rr = 1.0 + 0.3 * np.cos(5.0 * tt)
    return np.stack([rr * np.cos(tt), rr * np.sin(tt)], axis=1)


def fibonacci_sphere(n: int, seed: int, gen=None) -> np.ndarray:
    """Config 4: Fibonacci lattice plus 1e-3 seeded Gaussian jitter, projected
    back to the unit sphere."""
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    rho = np.sqrt(1.0 - z * z)
    f = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
    f = f + 1e-3 * _gen(gen).gaussian_matrix(n, 3, seed)
    return f / np.linalg.norm(f, axis=1, keepdims=True)


def make_points(name: str, n: int, gen=None) -> np.ndarray:
    g = _gen(gen)
    if name == "c1":
        return np.sort(g.random_cloud(n, 1, g.mix_seed(S0, 0xC1)), axis=0)
    if name == "c2":
        return np.sort(g.random_cloud(n, 1, g.mix_seed(S0, 0xC2)), axis=0)
    if name == "c3":
        return starfish_points(n, g.mix_seed(S0, 0xC3), gen)
    if name == "c4":
        return fibonacci_sphere(n, g.mix_seed(S0, 0xC4), gen)
    if name == "c5":
        return g.random_cloud(n, 3, g.mix_seed(S0, 0xC5))
    raise ValueError(name)


CONFIGS = {
    "c1": Workload("c1", 4096, 1, "log", True, 64, 20, 10,
                   description="1D N=4096 sorted U[0,1], explicit dense log|x-y| (A_ii=0), leaf 64, k=20, p=10"),
    "c2": Workload("c2", 65536, 1, "log", False, 64, 24, 10,
                   description="1D N=65536 U[0,1], on-the-fly log|x-y|, leaf 64, k=24, p=10"),
    "c3": Workload("c3", 262144, 2, "log", False, 128, 32, 10,
                   description="2D starfish N=262144 clustered, on-the-fly log|x-y|, quadtree leaf 128, k=32, p=10"),
    "c4": Workload("c4", 1 << 20, 3, "invdist4pi", False, 256, 48, 16,
                   description="3D Fibonacci sphere N=2^20, 1/(4 pi r), octree leaf 256, k=48, p=16"),
    "c5": Workload("c5", 1 << 19, 3, "exp", False, 256, 64, 16, param=0.1,
                   description="3D U[0,1]^3 N=2^19, exp(-r/0.1), octree leaf 256, k=64, p=16"),
}


def scaled(name: str, n: int) -> Workload:
    """Same generator and parameters at a smaller N (parity-test sizes)."""
    w = CONFIGS[name]
    return Workload(w.name, n, w.dim, w.kernel, w.dense, w.leaf, w.rank, w.oversample, w.param,
                    w.description + f" [scaled to N={n}]")
