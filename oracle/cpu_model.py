"""CPU reference timing for bench.py's reference arm -- TEST INFRASTRUCTURE ONLY.

The reference library cannot be built here (Eigen3 is absent, SURVEY.md
8(c)), so its CPU path is timed through this package's restatement of it
(hpeel_ref.compress: the reference's call pattern -- one dense test matrix
per color through the black box, serial per-pair QR / pseudo-inverse solves,
apply_truncated over all N rows, proj/src/peeling.cpp:158-275, :490-524).

* `timed_compress`: a full measured compress with per-phase wall seconds.
* `workload_counts`: exact column / flop counts of a workload from the
  oracle's own plans (tree, adjacency, colorings), in the reference's flop
  conventions (proj/include/hpeel/flops.hpp:18-20, proj/src/peeling.cpp:262-264,
  proj/src/linalg.cpp:116-117, proj/src/hmatrix.cpp:86-100).
* `apply_rate`: the black box's per-row cost, measured on a row subset of one
  dense test matrix of the full workload.
* `extrapolate`: full-workload seconds = measured apply rate x exact columns
  + per-flop rates of the other phases calibrated on a measured compress of a
  scaled instance x the full instance's flop counts (ranks taken as k).
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from . import hpeel_ref as R


def _threads(n):
    """threadpoolctl limits for BLAS (numpy/scipy) to n threads (None: all)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n) if n else threadpool_limits(limits=os.cpu_count())
    except ImportError:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


class ThreadedKernelOperator(R.KernelOperator):
    """KernelOperator whose row chunks run on a thread pool (numpy releases
    the GIL in the kernel evaluation and the chunk products): the "all host
    cores" variant of the on-the-fly black box. threads = 1 is the serial one."""

    def __init__(self, kind, points, param=0.1, threads=1, chunk=512):
        super().__init__(kind, points, param, chunk)
        self.threads = max(1, int(threads))

    def apply(self, x):
        n = self.shape[0]
        y = np.empty((n, x.shape[1]))
        starts = range(0, n, self.chunk)

        def work(i0):
            i1 = min(n, i0 + self.chunk)
            y[i0:i1] = self.block(i0, i1) @ x

        if self.threads == 1:
            for i0 in starts:
                work(i0)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(self.threads) as ex:
                list(ex.map(work, starts))
        return y

    apply_adjoint = apply


def make_operator(w, pts, threads=1):
    """The workload's black box in the oracle: the explicit dense matrix for
    config 1 (DenseOperator, BLAS threads), the on-the-fly kernel operator
    (row chunks on `threads` threads) otherwise."""
    if w.dense:
        same = np.eye(len(pts), dtype=bool)
        return R.DenseOperator(R.kernel_matrix(w.kernel, pts, pts, same, w.param))
    return ThreadedKernelOperator(w.kernel, pts, w.param, threads)


def timed_compress(w, pts, threads=None, seed=7):
    """Full oracle compress on `threads` BLAS threads (None: all): (seconds,
    per-phase seconds, rep, report)."""
    nthreads = threads or os.cpu_count() or 1
    # dense black box: BLAS threads; on-the-fly kernels: row chunks on threads
    # (BLAS single-threaded inside each chunk, no oversubscription)
    with _threads(nthreads if w.dense else 1):
        op = make_operator(w, pts, nthreads)
        t0 = time.perf_counter()
        tree = R.BoxTree(R.PointCloud(pts), w.leaf)
        times = R.PhaseTimes()
        times["tree"] = time.perf_counter() - t0
        rep, report = R.compress(op, tree, w.rank, w.oversample, seed, times=times)
        total = time.perf_counter() - t0
    return total, dict(times), rep, report


def _svd_flops(m, n):
    return 6 * m * n * n + 11 * n ** 3 if m >= n else 6 * n * m * m + 11 * m ** 3


def workload_counts(tree, adj, k, p, seed=7, ranks=None):
    """Exact black-box columns and reference flop counts of one compress.
    ranks: {(level, (a, b)): (ku, kv)} of a finished run, else k for all."""
    r = k + p
    cnt = lambda b: len(tree.box(b).points)  # noqa: E731
    out = {"h1_cols": 0, "leaf_cols": 0, "colors": {}, "qr": 0.0, "bsolve": 0.0, "peel": 0.0,
           "plan_s": 0.0, "n": tree.num_points}
    # apply_truncated(level) flops for one width-w product (hmatrix.cpp:86-100)
    trunc = [0.0] * (tree.depth + 1)
    acc = 0.0
    for l in range(2, tree.depth + 1):
        for a, b in R.admissible_pairs(tree, adj, l):
            ku, kv = ranks.get((l, (a, b)), (k, k)) if ranks else (k, k)
            acc += 2 * kv * cnt(b) + 2 * ku * kv + 2 * cnt(a) * ku
        trunc[l] = acc  # per unit width, levels 2..l
    for l in range(2, tree.depth + 1):
        pairs = R.admissible_pairs(tree, adj, l)
        if not pairs:
            continue
        t0 = time.perf_counter()
        plan = R.make_plan(tree, adj, l, R.H1, r, seed, 0)
        out["plan_s"] += time.perf_counter() - t0
        nc = sum(1 for m in plan.matrices if m.payload)
        out["colors"][l] = nc
        out["h1_cols"] += 2 * nc * r
        if l - 1 >= 2:
            out["peel"] += 2 * nc * r * trunc[l - 1]
        for a, b in pairs:
            ku, kv = ranks.get((l, (a, b)), (k, k)) if ranks else (k, k)
            ma, mb = cnt(a), cnt(b)
            out["qr"] += 2 * ma * r * r + 2 * mb * r * r
            f = 2 * r * r * ma + 2 * r * ku * ma + 2 * kv * r * mb
            if ku > 0:
                f += _svd_flops(r, ku) + 2 * ku * r * r
            if kv > 0:
                f += _svd_flops(r, kv) + 2 * kv * ku * r
            out["bsolve"] += f
    t0 = time.perf_counter()
    wl = tree.max_leaf_size()
    lplan = R.make_plan(tree, adj, tree.depth, R.LEAF, wl, seed, 0)
    out["plan_s"] += time.perf_counter() - t0
    nl = sum(1 for m in lplan.matrices if m.payload)
    out["colors"]["leaf"] = nl
    out["leaf_cols"] = nl * wl
    out["leaf_width"] = wl
    out["peel_leaf"] = nl * wl * trunc[tree.depth] if tree.depth >= 2 else 0.0
    return out


def apply_rate(w, pts, width, budget_s, threads=None):
    """Seconds per (row x test-matrix column) of the black box on the full
    point set: rows of one dense Gaussian test matrix pushed through the
    operator (the reference's per-color apply) until `budget_s` elapses."""
    n = len(pts)
    nthreads = threads or os.cpu_count() or 1
    op = make_operator(w, pts, nthreads)
    omega = np.random.default_rng(0).standard_normal((n, width))
    chunk = 256

    def rows(i0):
        i1 = min(n, i0 + chunk)
        if isinstance(op, R.DenseOperator):
            _ = op.a[i0:i1] @ omega
        else:
            _ = op.block(i0, i1) @ omega

    with _threads(1 if (nthreads > 1 and not w.dense) else threads):
        done, t0 = 0, time.perf_counter()
        if nthreads == 1 or w.dense:
            while done < n and time.perf_counter() - t0 < budget_s:
                rows(done)
                done = min(n, done + chunk)
        else:
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(nthreads) as ex:
                while done < n and time.perf_counter() - t0 < budget_s:
                    starts = list(range(done, min(n, done + chunk * nthreads), chunk))
                    list(ex.map(rows, starts))
                    done = min(n, done + chunk * nthreads)
        el = time.perf_counter() - t0
    return el / (done * width), done


def calibrate(w_scaled, pts_scaled, threads=None):
    """Per-unit costs of the non-apply phases from a measured compress of a
    scaled instance: seconds per reference flop (peel, QR, B) and the
    realize / plan overheads."""
    total, times, rep, _ = timed_compress(w_scaled, pts_scaled, threads)
    tree = rep.tree
    ranks = {(l, ab): (u.shape[1], v.shape[1]) for l in range(len(rep.levels)) for ab, (u, _, v) in rep.levels[l].items()}
    c = workload_counts(tree, rep.adj, w_scaled.rank, w_scaled.oversample, ranks=ranks)
    n = tree.num_points
    cols = c["h1_cols"] + c["leaf_cols"]
    rates = {
        "peel": (times.get("peel", 0.0) + times.get("leaf_peel", 0.0)) / max(c["peel"] + c["peel_leaf"], 1.0),
        "qr": times.get("qr", 0.0) / max(c["qr"], 1.0),
        "bsolve": times.get("bsolve", 0.0) / max(c["bsolve"], 1.0),
        "realize": (times.get("realize", 0.0) + times.get("leaf_realize", 0.0)) / max(n * cols, 1.0),
        "apply": (times.get("apply", 0.0) + times.get("leaf_apply", 0.0)) / max(n * cols, 1.0),
    }
    return {"total_s": total, "times": times, "counts": c, "rates": rates, "n": n}


def extrapolate(counts, apply_s_per_rowcol, cal):
    """Full-workload seconds per phase from exact counts, the measured apply
    rate and the calibrated per-flop rates."""
    n = counts["n"]
    cols = counts["h1_cols"] + counts["leaf_cols"]
    ph = {
        "apply": apply_s_per_rowcol * n * cols,
        "realize": cal["rates"]["realize"] * n * cols,
        "peel": cal["rates"]["peel"] * (counts["peel"] + counts["peel_leaf"]),
        "qr": cal["rates"]["qr"] * counts["qr"],
        "bsolve": cal["rates"]["bsolve"] * counts["bsolve"],
        "plan": counts["plan_s"],
    }
    ph["total"] = sum(ph.values())
    return ph


def dense_equivalent_flops(counts):
    """2 N^2 W of the reference's dense per-color applies."""
    n = counts["n"]
    return 2.0 * n * n * (counts["h1_cols"] + counts["leaf_cols"])


__all__ = ["timed_compress", "workload_counts", "apply_rate", "calibrate", "extrapolate",
           "dense_equivalent_flops", "make_operator"]

