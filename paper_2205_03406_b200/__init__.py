"""B200-native H1 graph-colored peeling core (arxiv 2205.03406).

Python surface mirroring the reference binding ``hpeel``
(proj/bindings/module.cpp:97-230): ``gaussian_matrix``, ``build_tree``,
``level_coloring``, ``dense_operator``, ``compress``, ``rel_error_power_method``
and the point generators, plus the on-the-fly kernel operators of
BASELINE.json. Every call goes through the C ABI of ``libhpeel_b200.so``; the
compression itself runs in hand-written sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, dptr, fmat, iptr, lptr, lib

__all__ = [
    "gaussian_matrix", "mix_seed", "random_cloud", "equispaced_1d", "uniform_grid_points",
    "BoxTree", "build_tree", "Plan", "plan", "level_coloring", "dsatur",
    "Operator", "dense_operator", "kernel_operator", "callback_operator", "CompressedRep", "compress",
    "compress_group", "shard_owners", "shard_memory_plan",
    "rel_error_power_method", "device_count", "debug_payload", "export_sizes", "pinned_empty",
    "load_rep", "save_dense_matrix", "load_dense_matrix",
]

MODES = {"h1": 0, "unif-stage1": 1, "unif-stage2": 2, "leaf": 3}
FORMATS = {"h1": 0, "unif-h1": 1, "h1-plus-unif": 2, "h2": 3}
STRATEGIES = {"graph": 0, "fallback-pattern": 1}
KERNELS = {"log": 1, "invdist4pi": 2, "exp": 3}


def device_count() -> int:
    n = C.c_int(0)
    check(lib().hp_device_count(C.byref(n)))
    return n.value


def launch_count() -> int:
    """Kernels launched by libhpeel_b200 so far in this process."""
    return int(lib().hp_launch_count())


def device_synchronize() -> None:
    check(lib().hp_device_synchronize())


def mix_seed(seed: int, *tags: int) -> int:
    for t in tags:
        seed = lib().hp_mix_seed(seed, t)
    return int(seed)


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """proj/src/rng.cpp:35-59 (row-major Box-Muller stream)."""
    out = np.zeros((rows, cols), dtype=np.float64, order="F")
    check(lib().hp_gaussian_matrix(rows, cols, seed, dptr(out)))
    return out


def random_cloud(n: int, dim: int, seed: int) -> np.ndarray:
    """proj/src/operators.cpp:88-95."""
    out = np.zeros((n, dim), dtype=np.float64, order="F")
    check(lib().hp_random_cloud(n, dim, seed, dptr(out)))
    return out


def equispaced_1d(n: int) -> np.ndarray:
    """proj/src/operators.cpp:97-103: (i + 0.5) / n."""
    return ((np.arange(n, dtype=np.float64) + 0.5) / float(n))[:, None]


def uniform_grid_points(per_dim: int, dim: int) -> np.ndarray:
    """proj/src/operators.cpp:74-86 (cell centers, dimension 0 fastest)."""
    total = per_dim ** dim
    idx = np.arange(total)
    out = np.empty((total, dim))
    for j in range(dim):
        out[:, j] = ((idx % per_dim).astype(np.float64) + 0.5) / float(per_dim)
        idx = idx // per_dim
    return out


class BoxTree:
    """BoxTree + AdjacencyInfo handle (binding PyTree, module.cpp:12-26)."""

    def __init__(self, handle, points: np.ndarray):
        self._h = C.c_void_p(handle)
        self.raw_points = points
        info = np.zeros(8, dtype=np.int64)
        check(lib().hp_tree_info(self._h, lptr(info)))
        (self.num_points, self.dim, self.depth, self.num_boxes, self.max_leaf_size,
         fp, self.leaf_capacity, self._npts) = (int(v) for v in info)
        self.fully_populated = bool(fp)
        self._boxes = None
        self._lists = {}

    def __del__(self):
        try:
            if self._h:
                lib().hp_tree_free(self._h)
        except Exception:
            pass

    def _box_arrays(self):
        if self._boxes is None:
            nb = self.num_boxes
            level = np.zeros(nb, dtype=np.int32)
            parent = np.zeros(nb, dtype=np.int32)
            coord = np.zeros((nb, self.dim), dtype=np.int64)
            off = np.zeros(nb + 1, dtype=np.int64)
            pts = np.zeros(max(self._npts, 1), dtype=np.int32)
            check(lib().hp_tree_boxes(self._h, iptr(level), iptr(parent), lptr(coord), lptr(off), iptr(pts)))
            self._boxes = (level, parent, coord, off, pts)
        return self._boxes

    def _list(self, which):
        if which not in self._lists:
            off = np.zeros(self.num_boxes + 1, dtype=np.int64)
            check(lib().hp_tree_lists(self._h, which, lptr(off), None))
            items = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
            check(lib().hp_tree_lists(self._h, which, lptr(off), iptr(items)))
            self._lists[which] = (off, items)
        return self._lists[which]

    def _get(self, which, box):
        off, items = self._list(which)
        return [int(v) for v in items[off[box]:off[box + 1]]]

    def level_boxes(self, level: int):
        lv = self._box_arrays()[0]
        return [int(i) for i in np.nonzero(lv == level)[0]]

    def box_level(self, box: int) -> int:
        return int(self._box_arrays()[0][box])

    def box_parent(self, box: int) -> int:
        return int(self._box_arrays()[1][box])

    def box_coord(self, box: int):
        return [int(v) for v in self._box_arrays()[2][box]]

    def box_points(self, box: int):
        off, pts = self._box_arrays()[3:]
        return pts[off[box]:off[box + 1]].tolist()

    def children(self, box: int):
        return self._get(4, box)

    def neighbors(self, box: int):
        return self._get(0, box)

    def interaction(self, box: int):
        return self._get(1, box)

    def coarse_leaf_neighbors(self, box: int):
        return self._get(2, box)

    def dense_partners(self, box: int):
        return self._get(3, box)

    @property
    def cross_level_adjacencies(self) -> int:
        return int(lib().hp_tree_cross_level_adjacencies(self._h))

    def _pairs(self, level):
        cache = self.__dict__.setdefault("_pair_cache", {})
        if level not in cache:
            cnt = C.c_int64(0)
            check(lib().hp_tree_pairs(self._h, level, C.byref(cnt), None))
            arr = np.zeros(max(2 * cnt.value, 2), dtype=np.int32)
            check(lib().hp_tree_pairs(self._h, level, C.byref(cnt), iptr(arr)))
            cache[level] = [(int(arr[2 * i]), int(arr[2 * i + 1])) for i in range(cnt.value)]
        return cache[level]  # shared: callers must not mutate

    def admissible_pairs(self, level: int):
        return self._pairs(level)

    def dense_pairs(self):
        return self._pairs(-1)

    def layout(self):
        """Device tree order: (perm, start, count)."""
        perm = np.zeros(self.num_points, dtype=np.int32)
        start = np.zeros(self.num_boxes, dtype=np.int64)
        count = np.zeros(self.num_boxes, dtype=np.int64)
        check(lib().hp_tree_layout(self._h, iptr(perm), lptr(start), lptr(count)))
        return perm, start, count


def build_tree(points, leaf_capacity: int) -> BoxTree:
    """PointCloud::from_raw + BoxTree::build + adjacency (module.cpp:19-26)."""
    pts = fmat(points)
    h = C.c_void_p()
    check(lib().hp_tree_build(dptr(pts), pts.shape[0], pts.shape[1], int(leaf_capacity), C.byref(h)))
    return BoxTree(h.value, pts)


class Plan:
    """make_plan output for one level (proj/src/peeling.cpp:98-154)."""

    def __init__(self, tree: BoxTree, level: int, mode: str, width: int, seed: int, phase: int,
                 pairwise: bool = False, strategy: str = "graph"):
        self.tree = tree
        self.width = width
        h = C.c_void_p()
        kind = 3 if strategy == "fallback-pattern" else int(pairwise)
        check(lib().hp_plan_build(tree._h, level, MODES[mode], width, seed, phase, kind, C.byref(h)))
        self._h = h
        self.pattern_map = None
        if kind == 3:
            cnt = C.c_int64(0)
            check(lib().hp_plan_block_map(h, C.byref(cnt), None))
            tri = np.zeros(max(3 * cnt.value, 3), dtype=np.int32)
            check(lib().hp_plan_block_map(h, C.byref(cnt), iptr(tri)))
            self.pattern_map = {(int(tri[3 * i]), int(tri[3 * i + 1])): int(tri[3 * i + 2]) for i in range(cnt.value)}
        info = np.zeros(8, dtype=np.int64)
        check(lib().hp_plan_info(h, lptr(info)))
        self.n_vertices, self.n_edges, self.n_colors, self.queue_ops = (int(v) for v in info[:4])
        npay, nzero, nown, nmp = (int(v) for v in info[4:])
        nv = self.n_vertices
        pay_off = np.zeros(nv + 1, dtype=np.int64)
        zero_off = np.zeros(nv + 1, dtype=np.int64)
        own_off = np.zeros(nv + 1, dtype=np.int64)
        pay_box = np.zeros(max(npay, 1), dtype=np.int32)
        pay_tag = np.zeros(max(npay, 1), dtype=np.int32)
        zero = np.zeros(max(nzero, 1), dtype=np.int32)
        owners = np.zeros(max(2 * nown, 2), dtype=np.int32)
        check(lib().hp_plan_sets(h, lptr(pay_off), iptr(pay_box), iptr(pay_tag), lptr(zero_off),
                                 iptr(zero), lptr(own_off), iptr(owners)))
        self.sets = []
        for i in range(nv):
            self.sets.append({
                "payload": [(int(pay_box[j]), int(pay_tag[j])) for j in range(pay_off[i], pay_off[i + 1])],
                "zero": [int(z) for z in zero[zero_off[i]:zero_off[i + 1]]],
                "owners": [(int(owners[2 * j]), int(owners[2 * j + 1])) for j in range(own_off[i], own_off[i + 1])],
            })
        goff = np.zeros(nv + 1, dtype=np.int64)
        check(lib().hp_plan_graph(h, lptr(goff), None))
        gadj = np.zeros(max(int(goff[-1]), 1), dtype=np.int32)
        check(lib().hp_plan_graph(h, lptr(goff), iptr(gadj)))
        self.edges = [[int(w) for w in gadj[goff[v]:goff[v + 1]]] for v in range(nv)]
        color = np.zeros(max(nv, 1), dtype=np.int32)
        dcolor = np.zeros(max(nv, 1), dtype=np.int32)
        dn = C.c_int(0)
        check(lib().hp_plan_coloring(h, iptr(color), iptr(dcolor), C.byref(dn)))
        self.color = [int(c) for c in color[:nv]]
        self.dsatur_color = [int(c) for c in dcolor[:nv]]
        self.dsatur_colors = dn.value
        moff = np.zeros(self.n_colors + 1, dtype=np.int64)
        mbox = np.zeros(max(nmp, 1), dtype=np.int32)
        if nv or self.pattern_map is not None:
            check(lib().hp_plan_matrices(h, lptr(moff), iptr(mbox)))
        self.color_payload = [[int(b) for b in mbox[moff[c]:moff[c + 1]]] for c in range(self.n_colors)]

    def __del__(self):
        try:
            lib().hp_plan_free(self._h)
        except Exception:
            pass

    def block_to_matrix(self):
        if self.pattern_map is not None:
            return dict(self.pattern_map)
        out = {}
        for i, s in enumerate(self.sets):
            for o in s["owners"]:
                out[o] = self.color[i]
        return out

    def realize(self, color: int) -> np.ndarray:
        out = np.zeros((self.tree.num_points, self.width), order="F")
        check(lib().hp_plan_realize(self._h, color, dptr(out)))
        return out


def plan(tree, level, mode="h1", width=10, seed=0, phase=0, pairwise=False, implicit=False) -> Plan:
    """`pairwise`: literal O(V^2) graph scan; `implicit`: the driver's graph-free
    DSatur (no edge lists: plan.graph() is empty)."""
    return Plan(tree, level, mode, width, seed, phase, 2 if implicit else pairwise)


def level_coloring(tree: BoxTree, level: int, mode: str) -> dict:
    """module.cpp:190-205."""
    p = Plan(tree, level, mode, 1, 0, 0)
    return {"n_vertices": p.n_vertices, "n_edges": p.n_edges, "n_colors": p.n_colors}


def dsatur(edges):
    """DSatur (proj/src/coloring.cpp:169-216) on an explicit adjacency list."""
    nv = len(edges)
    off = np.zeros(nv + 1, dtype=np.int64)
    for v, e in enumerate(edges):
        off[v + 1] = off[v] + len(e)
    adj = np.array([w for e in edges for w in sorted(e)] or [0], dtype=np.int32)
    color = np.zeros(max(nv, 1), dtype=np.int32)
    nc = C.c_int(0)
    qops = C.c_int64(0)
    check(lib().hp_dsatur(nv, lptr(off), iptr(adj), iptr(color), C.byref(nc), C.byref(qops)))
    return {"color": [int(c) for c in color[:nv]], "num_colors": nc.value, "queue_ops": qops.value}


class Operator:
    """Device-resident black box (LinearOperator, linear_operator.hpp:12-24)."""

    def __init__(self, handle, n):
        self._h = C.c_void_p(handle)
        self.shape = (n, n)

    def __del__(self):
        try:
            lib().hp_op_free(self._h)
        except Exception:
            pass

    def _apply(self, x, adjoint):
        x = fmat(x)
        y = np.zeros_like(x, order="F")
        check(lib().hp_op_apply(self._h, int(adjoint), dptr(x), x.shape[1], dptr(y)))
        return y

    def apply(self, x):
        return self._apply(x, False)

    def apply_adjoint(self, x):
        return self._apply(x, True)


def dense_operator(a, device: int = 0) -> Operator:
    a = fmat(a)
    h = C.c_void_p()
    check(lib().hp_op_dense(dptr(a), a.shape[0], device, C.byref(h)))
    return Operator(h.value, a.shape[0])


class CallbackOperator(Operator):
    """A Python black box behind the C ABI's callback boundary (hp_op_callback:
    the reference's virtual LinearOperator::apply / apply_adjoint,
    proj/include/hpeel/linear_operator.hpp:19-20). `apply(x, adjoint)` gets an
    n x w float64 array in the caller's point order and returns A x (A^T x).
    Exceptions raised inside are re-raised by the next compress()."""

    def __init__(self, n: int, apply, symmetric: bool = True, device: int = 0):
        self._fn = apply
        self.error = None
        self.calls = 0
        self.columns = [0, 0]

        def trampoline(ctx, adjoint, x, w, y, stream):
            try:
                xa = np.ctypeslib.as_array(x, shape=(int(n) * int(w),)).reshape((n, w), order="F")
                out = np.asarray(self._fn(xa, bool(adjoint)), dtype=np.float64)
                if out.shape != (n, w):
                    raise ValueError(f"black box returned shape {out.shape}, expected {(n, w)}")
                ya = np.ctypeslib.as_array(y, shape=(int(n) * int(w),)).reshape((n, w), order="F")
                ya[...] = out
                self.calls += 1
                self.columns[int(bool(adjoint))] += int(w)
                return 0
            except BaseException as e:  # noqa: BLE001 -- reported through compress()
                self.error = e
                return 1

        self._cb = _lib.APPLY_FN(trampoline)  # kept alive with the operator
        h = C.c_void_p()
        check(lib().hp_op_callback(int(n), int(bool(symmetric)), 0, C.cast(self._cb, C.c_void_p), None, device,
                                   C.byref(h)))
        super().__init__(h.value, n)


def callback_operator(n: int, apply, symmetric: bool = True, device: int = 0) -> CallbackOperator:
    """Black box from a Python function apply(x, adjoint) -> y (host arrays)."""
    return CallbackOperator(n, apply, symmetric, device)


def kernel_operator(kind: str, points, param: float = 1.0, device: int = 0) -> Operator:
    """On-the-fly kernel black box over raw coordinates (BASELINE.json configs)."""
    pts = fmat(points)
    h = C.c_void_p()
    check(lib().hp_op_kernel(KERNELS[kind], dptr(pts), pts.shape[0], pts.shape[1], float(param), device, C.byref(h)))
    return Operator(h.value, pts.shape[0])


class CompressedRep:
    """Device-resident H1Rep (hmatrix.hpp:52-70) + RunReport."""

    def __init__(self, handle, tree: BoxTree, rank: int, oversample: int):
        self._h = C.c_void_p(handle)
        self.tree = tree
        self.rank = rank
        self.width = rank + oversample
        self.format = "h1"
        totals = np.zeros(9)
        nph = C.c_int64(0)
        check(lib().hp_rep_report(self._h, dptr(totals), C.byref(nph)))
        ln = C.c_int64(0)
        check(lib().hp_rep_csv(self._h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        check(lib().hp_rep_csv(self._h, buf, ln.value + 1, C.byref(ln)))
        phases = []
        for i in range(nph.value):
            ints = np.zeros(7, dtype=np.int64)
            times = np.zeros(13)
            check(lib().hp_rep_phase(self._h, i, lptr(ints), dptr(times)))
            phases.append({
                "phase": "leaf" if ints[0] else "h1", "level": int(ints[1]), "colors": int(ints[2]),
                "forward_cols": int(ints[3]), "adjoint_cols": int(ints[4]), "net_flops": int(ints[5]),
                "apply_path": "int8" if ints[6] else "fp64",
                "wall_ms_total": times[0], "wall_ms_net": times[1], "apply_ms": times[2],
                "peel_ms": times[3], "qr_ms": times[4], "bsolve_ms": times[5],
                "apply_flops": times[6], "kernel_evals": times[7], "host_wait_ms": times[8],
                "start_ms": times[9], "peel_flops": times[10], "qr_flops": times[11], "bsolve_flops": times[12],
            })
        self.report = {
            "forward_cols": int(totals[0]), "adjoint_cols": int(totals[1]),
            "max_sampling_colors": int(totals[2]), "wall_s_total": totals[3],
            "wall_s_net": totals[4], "net_flops": int(totals[5]), "setup_ms": totals[6],
            "peak_device_bytes": totals[7], "exchange_bytes": totals[8],
            "csv": buf.value.decode(),
            "phases": phases,
        }

    def __del__(self):
        try:
            lib().hp_rep_free(self._h)
        except Exception:
            pass

    def _apply(self, x, adjoint):
        x = fmat(x)
        y = np.zeros_like(x, order="F")
        check(lib().hp_rep_apply(self._h, int(adjoint), dptr(x), x.shape[1], dptr(y)))
        return y

    def apply(self, x):
        return self._apply(x, False)

    def apply_adjoint(self, x):
        return self._apply(x, True)

    def num_pairs(self, level: int) -> int:
        c = C.c_int64(0)
        check(lib().hp_rep_num_pairs(self._h, level, C.byref(c)))
        return c.value

    def block(self, level: int, pair: int):
        """(U, B, V) of admissible_pairs(level)[pair], rows in box.points order."""
        ku, kv = C.c_int(0), C.c_int(0)
        check(lib().hp_rep_block(self._h, level, pair, C.byref(ku), C.byref(kv), None, None, None))
        a, b = self.tree.admissible_pairs(level)[pair]
        ma, mb = len(self.tree.box_points(a)), len(self.tree.box_points(b))
        u = np.zeros((ma, ku.value), order="F")
        bb = np.zeros((ku.value, kv.value), order="F")
        v = np.zeros((mb, kv.value), order="F")
        check(lib().hp_rep_block(self._h, level, pair, C.byref(ku), C.byref(kv), dptr(u), dptr(bb), dptr(v)))
        return u, bb, v

    def dense_block(self, pair: int) -> np.ndarray:
        lam, mu = self.tree.dense_pairs()[pair]
        d = np.zeros((len(self.tree.box_points(lam)), len(self.tree.box_points(mu))), order="F")
        check(lib().hp_rep_dense_block(self._h, pair, dptr(d)))
        return d

    def captured(self, level: int, pair: int) -> np.ndarray:
        """Post-peel samples [Y | Z] of a pair (level < 0: leaf probe block)."""
        rows, cols = C.c_int64(0), C.c_int64(0)
        check(lib().hp_rep_captured(self._h, level, pair, C.byref(rows), C.byref(cols), None))
        out = np.zeros((rows.value, cols.value), order="F")
        check(lib().hp_rep_captured(self._h, level, pair, C.byref(rows), C.byref(cols), dptr(out)))
        return out

    def shard(self):
        """(world, rank) of the group that built this representation."""
        w, r = C.c_int(0), C.c_int(0)
        check(lib().hp_rep_shard(self._h, 0, 0, C.byref(w), C.byref(r), None))
        return w.value, r.value

    def holds(self, level: int, pair: int) -> bool:
        """Whether this rank holds block `pair` of `level` (level < 0: dense block)."""
        h = C.c_int(0)
        check(lib().hp_rep_shard(self._h, int(level), int(pair), None, None, C.byref(h)))
        return bool(h.value)

    def captured_raw(self, level: int, pair: int) -> np.ndarray:
        """The same block before peeling: rows of A Omega | A^T Psi."""
        rows, cols = C.c_int64(0), C.c_int64(0)
        check(lib().hp_rep_captured_raw(self._h, level, pair, C.byref(rows), C.byref(cols), None))
        out = np.zeros((rows.value, cols.value), order="F")
        check(lib().hp_rep_captured_raw(self._h, level, pair, C.byref(rows), C.byref(cols), dptr(out)))
        return out

    def storage(self) -> dict:
        t = C.c_int64(0)
        check(lib().hp_rep_storage(self._h, C.byref(t)))
        return {"total": t.value, "per_dof": t.value / float(self.tree.num_points)}

    def sizes(self):
        f, d = C.c_int64(0), C.c_int64(0)
        check(lib().hp_rep_sizes(self._h, C.byref(f), C.byref(d)))
        return f.value, d.value

    def save(self, path: str) -> None:
        """save_rep (proj/src/serialize.cpp:156-188): the reference's .hrep file."""
        check(lib().hp_rep_save(self._h, str(path).encode()))

    def export(self, host_factors: np.ndarray, host_dense: np.ndarray) -> int:
        """Bulk device->host copy of the whole representation; returns bytes."""
        b = C.c_int64(0)
        check(lib().hp_rep_export(self._h, dptr(host_factors), dptr(host_dense), C.byref(b)))
        return b.value


class Comm:
    """NCCL communicator of one rank (one process per GPU)."""

    def __init__(self, unique_id: bytes, rank: int, world: int, device: int = 0):
        h = C.c_void_p()
        check(lib().hp_comm_create(unique_id, int(rank), int(world), int(device), C.byref(h)))
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().hp_comm_unique_id(buf))
        return buf.raw

    def __del__(self):
        try:
            lib().hp_comm_free(self._h)
        except Exception:
            pass


def partition_ranges(work, world: int):
    """Contiguous work-balanced ranges every rank computes identically."""
    work = np.ascontiguousarray(work, dtype=np.float64)
    out = np.zeros(world + 1, dtype=np.int64)
    check(lib().hp_partition_ranges(dptr(work), work.size, int(world), lptr(out)))
    return [int(v) for v in out]


def _raise_callback(op, exc):
    err = getattr(op, "error", None)
    if err is not None:
        op.error = None
        raise err from exc
    raise exc


def compress(op: Operator, tree: BoxTree, format: str = "h1", rank: int = 10, oversample: int = 10,
             tol: float = 0.0, seed: int = 0, strategy: str = "graph", capture: bool = False,
             comm: "Comm | None" = None, export_to=None) -> CompressedRep:
    """compress_py (module.cpp:65-93) on the device; fixed-rank H1 only.
    `comm`: this process's rank of an NCCL group (owner-computes sharding:
    the representation holds the factors of the pairs touching this rank's
    boxes).
    `export_to=(host_factors, host_dense)`: float64 arrays of export_sizes()
    filled with the representation while it is built (each level as soon as
    it is final; asynchronous when they come from pinned_empty())."""
    if format not in FORMATS:
        raise ValueError("unknown format: " + format)
    if strategy not in STRATEGIES:
        raise ValueError("unknown strategy: " + strategy)
    if tol > 0.0:
        raise ValueError("relative-tolerance truncation is outside the H1 fixed-rank hot path")
    h = C.c_void_p()
    if export_to is not None:
        if capture:
            raise ValueError("export_to cannot be combined with capture")
        hf, hd = export_to
        for a in (hf, hd):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
                raise ValueError("export arrays must be contiguous float64")
        try:
            check(lib().hp_compress_export(op._h, tree._h, int(rank), int(oversample), int(seed), FORMATS[format],
                                           STRATEGIES[strategy], comm._h if comm else None, dptr(hf), hf.size,
                                           dptr(hd), hd.size, C.byref(h)))
        except (RuntimeError, ValueError, AssertionError) as e:
            _raise_callback(op, e)
        return CompressedRep(h.value, tree, rank, oversample)
    try:
        check(lib().hp_compress_ex(op._h, tree._h, int(rank), int(oversample), int(seed), FORMATS[format],
                                   STRATEGIES[strategy], int(capture), comm._h if comm else None, C.byref(h)))
    except (RuntimeError, ValueError, AssertionError) as e:
        _raise_callback(op, e)
    return CompressedRep(h.value, tree, rank, oversample)


def compress_group(op: Operator, tree: BoxTree, world: int, rank: int = 10, oversample: int = 10, seed: int = 0,
                   capture: bool = False) -> list:
    """compress() on `world` ranks emulated by threads of this process on the
    operator's device: the owner-computes sharded path with device copies in
    place of NCCL. Returns one representation per rank."""
    hs = (C.c_void_p * int(world))()
    try:
        check(lib().hp_compress_group(op._h, tree._h, int(rank), int(oversample), int(seed), 0, 0, int(capture),
                                      int(world), hs))
    except (RuntimeError, ValueError, AssertionError) as e:
        _raise_callback(op, e)
    return [CompressedRep(hs[g], tree, rank, oversample) for g in range(int(world))]


def shard_owners(tree: BoxTree, world: int):
    """(owner per box (-1 above the cut), cut level, rank point bounds)."""
    owner = np.zeros(tree.num_boxes, dtype=np.int32)
    cut = C.c_int(0)
    bounds = np.zeros(int(world) + 1, dtype=np.int64)
    check(lib().hp_shard_owners(tree._h, int(world), iptr(owner), C.byref(cut), lptr(bounds)))
    return owner, cut.value, bounds


def shard_exchange_counts(tree: BoxTree, rank: int, world: int, shard: int, level: int, phase: int):
    """(send[world], recv[world]) doubles of shard `shard`'s crossing-pair
    exchange `phase` (1: V, 2: U and B) at `level`."""
    send = np.zeros(int(world), dtype=np.int64)
    recv = np.zeros(int(world), dtype=np.int64)
    check(lib().hp_shard_exchange_counts(tree._h, int(rank), int(world), int(shard), int(level), int(phase),
                                         lptr(send), lptr(recv)))
    return send, recv


def shard_memory_plan(tree: BoxTree, rank: int, oversample: int, world: int) -> np.ndarray:
    """Per-rank device bytes (world x 4): factors held, dense blocks, largest
    level's samples + apply buffers, total estimate."""
    out = np.zeros(int(world) * 4)
    check(lib().hp_shard_memory_plan(tree._h, int(rank), int(oversample), int(world), dptr(out)))
    return out.reshape(int(world), 4)


def load_rep(path: str, device: int = 0) -> "CompressedRep":
    """load_rep (proj/src/serialize.cpp:190-250) onto `device`; H1 files only.
    The representation's embedded tree is `rep.tree` (no point coordinates)."""
    h, t = C.c_void_p(), C.c_void_p()
    check(lib().hp_rep_load(str(path).encode(), int(device), C.byref(h), C.byref(t)))
    tree = BoxTree(t.value, None)
    return CompressedRep(h.value, tree, 1, 0)


def save_dense_matrix(path: str, a) -> None:
    """save_dense_matrix (serialize.cpp:252-256): "HPEELDM1" + matrix."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    check(lib().hp_save_dense_matrix(str(path).encode(), dptr(a), a.shape[0], a.shape[1]))


def load_dense_matrix(path: str) -> np.ndarray:
    """load_dense_matrix (serialize.cpp:258-264)."""
    rows, cols = C.c_int64(0), C.c_int64(0)
    check(lib().hp_load_dense_matrix(str(path).encode(), C.byref(rows), C.byref(cols), None, 0))
    out = np.zeros((rows.value, cols.value), order="F")
    check(lib().hp_load_dense_matrix(str(path).encode(), None, None, dptr(out), out.size))
    return out


def export_sizes(tree: BoxTree, rank: int, world: int = 1, shard: int = 0):
    """(factor doubles, dense doubles) of the host arrays ``compress(...,
    export_to=...)`` and ``CompressedRep.export`` fill for this tree and rank
    (of shard `shard` of a `world`-rank group)."""
    f, d = C.c_int64(0), C.c_int64(0)
    if world == 1:
        check(lib().hp_export_sizes(tree._h, int(rank), C.byref(f), C.byref(d)))
    else:
        check(lib().hp_export_sizes_shard(tree._h, int(rank), int(world), int(shard), C.byref(f), C.byref(d)))
    return f.value, d.value


class _PinnedBlock:
    def __init__(self, nbytes):
        self.ptr = C.c_void_p()
        check(lib().hp_host_alloc(int(nbytes), C.byref(self.ptr)))
        self.nbytes = int(nbytes)

    def __del__(self):
        if self.ptr and _lib._lib is not None:
            _lib._lib.hp_host_free(self.ptr)
            self.ptr = None


def pinned_empty(n: int) -> np.ndarray:
    """float64 array of n elements in page-locked host memory (cudaHostAlloc),
    so device->host exports run asynchronously at full link speed."""
    blk = _PinnedBlock(max(int(n), 1) * 8)
    buf = (C.c_double * max(int(n), 1)).from_address(blk.ptr.value)
    arr = np.frombuffer(buf, dtype=np.float64, count=int(n))
    buf._hp_block = blk  # every view's base chain ends at buf: freed with the last view
    return arr


def rel_error_power_method(rep: CompressedRep, ref: Operator, iters: int = 20, seed: int = 0) -> float:
    """proj/src/linalg.cpp:206-218 (module.cpp:219-229)."""
    out = C.c_double(0.0)
    try:
        check(lib().hp_rel_error_power_method(rep._h, ref._h, int(iters), int(seed), C.byref(out)))
    except (RuntimeError, ValueError, AssertionError) as e:
        _raise_callback(ref, e)
    return out.value


def set_k2_mode(mode: int) -> None:
    """K2 probe bits (probe header): 16 = FP64 apply with the payload chunks in
    reverse order (another summation order, results valid); 8 = checked
    evaluation path, 4 = fused kernel (results identical); 1 / 2 skip work
    (invalid results, timing only)."""
    lib().hp_debug_set_k2_mode(int(mode))


def set_k2_path(path: str) -> None:
    """Black-box apply arithmetic: "int8" (default: exact fixed-point digit
    products on the int8 tensor cores wherever eligible) or "fp64" (FP64
    DMMA for every apply). For A/B parity tests and measurements."""
    lib().hp_debug_set_k2_path({"int8": 0, "fp64": 1, "int8-nomma": 2, "int8-noeval": 3, "int8-mma2": 5,
                                 "int8-noeval-mma2": 7,
                                 "int8-nodsmem": 9, "int8-noeval-nodsmem": 11}[path])


def debug_log(x, device: int = 0) -> np.ndarray:
    """Device log used by the log-kernel black box (accuracy probe)."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    out = np.zeros_like(x)
    check(lib().hp_debug_log(dptr(x), x.size, device, dptr(out)))
    return out


def debug_qr(blocks, kmax: int, device: int = 0):
    """K4 probe: batched range finder (pivoted QR, keep rule, Q(:, :kmax)) of
    equal-width blocks. Returns ([Q_i], ranks, device_ms)."""
    blocks = [np.asarray(b, dtype=np.float64) for b in blocks]
    if not blocks:
        return [], np.zeros(0, dtype=np.int32), 0.0
    cols = blocks[0].shape[1]
    rows = np.array([b.shape[0] for b in blocks], dtype=np.int32)
    flat = np.concatenate([np.asfortranarray(b).ravel(order="F") for b in blocks])
    q = np.zeros(int((rows.astype(np.int64) * kmax).sum()))
    ranks = np.zeros(len(blocks), dtype=np.int32)
    ms = C.c_double(0.0)
    check(lib().hp_debug_qr(dptr(flat), iptr(rows), len(blocks), cols, kmax, device, dptr(q),
                            iptr(ranks), C.byref(ms)))
    out, o = [], 0
    for m in rows:
        out.append(q[o:o + m * kmax].reshape((m, kmax), order="F"))
        o += m * kmax
    return out, ranks, ms.value


def debug_payload(tree: BoxTree, level: int, r: int, seed: int, device: int = 0) -> np.ndarray:
    """K1 probe: n x 2r payload rows (input order) generated on the device."""
    out = np.zeros((tree.num_points, 2 * r), order="F")
    check(lib().hp_debug_payload(tree._h, level, r, seed, device, dptr(out)))
    return out
