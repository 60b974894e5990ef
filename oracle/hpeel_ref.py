"""Reference restatement of the hpeel H1 path (see oracle/__init__.py).

TEST INFRASTRUCTURE ONLY: never imported by the product package.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

__all__ = [
    "GAMMA", "scramble", "mix_seed", "SplitMix64", "gaussian_matrix", "gaussian_matrix_libm",
    "random_cloud", "equispaced_1d", "uniform_grid_points", "PointCloud", "Box", "BoxTree",
    "Adjacency", "adjacency", "admissible_pairs", "dense_pairs", "ConstraintSet",
    "build_constraints", "incompatible", "build_graph", "build_graph_literal", "dsatur_color", "plan_coloring",
    "BlockTestMatrix", "payload_gaussian", "assemble_test_matrices", "make_plan",
    "qr_orthonormal", "pinv_apply", "DenseOperator", "KernelOperator", "H1Rep", "run_h1",
    "extract_leaf", "compress", "rel_error_power_method", "synth_rank_structured",
    "kernel_matrix", "PhaseTimes", "H1", "LEAF", "UNIF2", "BASIS", "UnifH1Rep", "run_uniform", "UNIF1", "save_rep_bytes", "load_rep_bytes", "save_dense_matrix_bytes",
    "REP_MAGIC", "DENSE_MAGIC",
]

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
H1, UNIF1, UNIF2, LEAF = 0, 1, 2, 3
GAUSSIAN, IDENTITY, BASIS = 0, 1, 2


# --------------------------------------------------------------------------- RNG
# proj/src/rng.cpp:8-59, proj/include/hpeel/rng.hpp:12-48

def scramble(z: int) -> int:
    """proj/src/rng.cpp:11-15."""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix_seed(seed: int, *tags: int) -> int:
    """proj/src/rng.cpp:31-33 and the variadic form rng.hpp:39-42."""
    for t in tags:
        seed = scramble((seed * GAMMA + t + 1) & M64)
    return seed


class SplitMix64:
    """proj/src/rng.cpp:18-29."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + GAMMA) & M64
        return scramble(self.state)

    def next_open_closed(self) -> float:
        return float((self.next() >> 11) + 1) * 2.0 ** -53

    def next_closed_open(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53


def _scramble_np(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _uniform_pairs(seed: int, npairs: int):
    q = np.arange(npairs, dtype=np.uint64)
    s = np.uint64(seed & M64)
    g = np.uint64(GAMMA)
    with np.errstate(over="ignore"):
        z1 = _scramble_np(s + (np.uint64(2) * q + np.uint64(1)) * g)
        z2 = _scramble_np(s + (np.uint64(2) * q + np.uint64(2)) * g)
    u1 = ((z1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (z2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return u1, u2


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """proj/src/rng.cpp:35-59: row-major Box-Muller stream, the sine variate
    of each (u1, u2) pair is the next entry. Vectorized; log/cos/sin from
    numpy (within an ulp of glibc, see gaussian_matrix_libm)."""
    if rows < 0 or cols < 0:
        raise ValueError("negative shape")
    total = rows * cols
    npairs = (total + 1) // 2
    u1, u2 = _uniform_pairs(seed, npairs)
    radius = np.sqrt(-2.0 * np.log(u1))
    angle = 2.0 * math.pi * u2
    out = np.empty(2 * npairs)
    out[0::2] = radius * np.cos(angle)
    out[1::2] = radius * np.sin(angle)
    return out[:total].reshape(rows, cols)


def gaussian_matrix_libm(rows: int, cols: int, seed: int) -> np.ndarray:
    """Same stream, scalar loop with the C library's log/cos/sin (the
    reference's std::log/std::cos/std::sin), for bit-exact pinning."""
    st = SplitMix64(seed)
    out = np.empty((rows, cols))
    spare, have = 0.0, False
    for i in range(rows):
        for j in range(cols):
            if have:
                out[i, j] = spare
                have = False
                continue
            u1 = st.next_open_closed()
            u2 = st.next_closed_open()
            radius = math.sqrt(-2.0 * math.log(u1))
            angle = 2.0 * math.pi * u2
            out[i, j] = radius * math.cos(angle)
            spare = radius * math.sin(angle)
            have = True
    return out


def random_cloud(n: int, dim: int, seed: int) -> np.ndarray:
    """proj/src/operators.cpp:88-95 (row by row, next_closed_open)."""
    u1, _ = None, None
    total = n * dim
    q = np.arange(1, total + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _scramble_np(np.uint64(seed & M64) + q * np.uint64(GAMMA))
    vals = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return vals.reshape(n, dim)


def equispaced_1d(n: int) -> np.ndarray:
    """proj/src/operators.cpp:97-103."""
    return ((np.arange(n, dtype=np.float64) + 0.5) / float(n))[:, None]


def uniform_grid_points(per_dim: int, dim: int) -> np.ndarray:
    """proj/src/operators.cpp:74-86."""
    total = per_dim ** dim
    out = np.empty((total, dim))
    rem = np.arange(total)
    for j in range(dim):
        out[:, j] = ((rem % per_dim).astype(np.float64) + 0.5) / float(per_dim)
        rem = rem // per_dim
    return out


# --------------------------------------------------------------------------- tree
# proj/src/box_tree.cpp

class PointCloud:
    """proj/src/box_tree.cpp:55-70."""

    def __init__(self, raw):
        raw = np.asarray(raw, dtype=np.float64)
        if raw.ndim == 1:
            raw = raw[:, None]
        if raw.shape[0] < 1:
            raise ValueError("empty point cloud")
        if not np.all(np.isfinite(raw)):
            raise ValueError("non-finite coordinates")
        c = raw.copy()
        for j in range(raw.shape[1]):
            lo, hi = raw[:, j].min(), raw[:, j].max()
            c[:, j] = (raw[:, j] - lo) / (hi - lo) if hi > lo else 0.5
        self.coords = c

    @property
    def dim(self):
        return self.coords.shape[1]

    def __len__(self):
        return self.coords.shape[0]


@dataclass
class Box:
    id: int
    level: int
    coord: tuple
    parent: int
    children: list = field(default_factory=list)
    points: np.ndarray = None

    @property
    def is_leaf(self):
        return not self.children


class BoxTree:
    """BoxTree::build, proj/src/box_tree.cpp:99-180 (BFS ids; split boxes with
    more than m points; children in corner-mask order; a point on a bisection
    plane goes to the lower child)."""

    MAX_DEPTH = 62

    def __init__(self, cloud: PointCloud, leaf_capacity: int):
        if leaf_capacity < 1:
            raise ValueError("leaf capacity >= 1")
        d = cloud.dim
        self.dim = d
        self.leaf_capacity = leaf_capacity
        self.num_points = len(cloud)
        self.boxes = [Box(0, 0, tuple([0] * d), -1, [], np.arange(len(cloud)))]
        self.levels = [[0]]
        frontier = [0]
        level = 0
        while True:
            if not any(len(self.boxes[i].points) > leaf_capacity for i in frontier):
                break
            if level >= self.MAX_DEPTH:
                raise RuntimeError("degenerate geometry: leaf capacity unreachable at depth cap")
            nxt = []
            for bid in frontier:
                parent = self.boxes[bid]
                if len(parent.points) <= leaf_capacity:
                    continue
                pts = parent.points
                mask = np.zeros(len(pts), dtype=np.int64)
                for j in range(d):
                    lo = math.ldexp(float(parent.coord[j]), -parent.level)
                    hi = math.ldexp(float(parent.coord[j] + 1), -parent.level)
                    mid = 0.5 * (lo + hi)
                    mask |= (cloud.coords[pts, j] > mid).astype(np.int64) << j
                for m in range(1 << d):
                    sel = pts[mask == m]
                    if len(sel) == 0:
                        continue
                    cid = len(self.boxes)
                    coord = tuple(2 * parent.coord[j] + ((m >> j) & 1) for j in range(d))
                    self.boxes.append(Box(cid, level + 1, coord, bid, [], sel))
                    parent.children.append(cid)
                    nxt.append(cid)
            self.levels.append(nxt)
            frontier = nxt
            level += 1
        self.depth = level

    def level_boxes(self, level):
        return self.levels[level]

    def box(self, i):
        return self.boxes[i]

    @property
    def num_boxes(self):
        return len(self.boxes)

    def max_leaf_size(self):
        return max(len(b.points) for b in self.boxes if b.is_leaf)

    def is_fully_populated(self):
        want = 1 << self.dim
        return all(len(b.children) == want for b in self.boxes if b.level < self.depth)


@dataclass
class Adjacency:
    neighbors: list
    interaction: list
    coarse_leaf_neighbors: list
    dense_partners: list
    cross_level_adjacencies: int


def adjacency(tree: BoxTree) -> Adjacency:
    """proj/src/box_tree.cpp:214-300."""
    nb = tree.num_boxes
    d = tree.dim
    index = [dict() for _ in range(tree.depth + 1)]
    for b in tree.boxes:
        index[b.level][b.coord] = b.id
    neighbors = [None] * nb
    offsets = [()]
    for _ in range(d):
        offsets = [o + (s,) for o in offsets for s in (-1, 0, 1)]
    for b in tree.boxes:
        lim = (1 << b.level) - 1
        ns = []
        for off in offsets:
            probe = tuple(b.coord[j] + off[j] for j in range(d))
            if all(0 <= p <= lim for p in probe) and probe in index[b.level]:
                ns.append(index[b.level][probe])
        neighbors[b.id] = sorted(ns)
    interaction = [[] for _ in range(nb)]
    for b in tree.boxes:
        if b.parent < 0:
            continue
        il = []
        for pn in neighbors[b.parent]:
            for c in tree.boxes[pn].children:
                cc = tree.boxes[c].coord
                if any(abs(cc[j] - b.coord[j]) > 1 for j in range(d)):
                    il.append(c)
        interaction[b.id] = sorted(il)
    cl = [[] for _ in range(nb)]
    cross = 0
    for b in tree.boxes:
        if b.parent < 0:
            continue
        s = set(cl[b.parent])
        s.update(pn for pn in neighbors[b.parent] if tree.boxes[pn].is_leaf)
        cl[b.id] = sorted(s)
        cross += len(cl[b.id])
    dp = [set() for _ in range(nb)]
    for b in tree.boxes:
        if not b.is_leaf:
            continue
        dp[b.id].update(n for n in neighbors[b.id] if tree.boxes[n].is_leaf)
        for c in cl[b.id]:
            dp[b.id].add(c)
            dp[c].add(b.id)
    return Adjacency(neighbors, interaction, cl, [sorted(s) for s in dp], cross)


def admissible_pairs(tree, adj, level):
    """proj/src/box_tree.cpp:302-313."""
    if level < 2 or level > tree.depth:
        raise ValueError("admissible pairs exist for levels 2..depth")
    return [(a, b) for a in tree.level_boxes(level) for b in adj.interaction[a]]


def dense_pairs(tree, adj):
    """proj/src/box_tree.cpp:315-323."""
    return [(b.id, m) for b in tree.boxes if b.is_leaf for m in adj.dense_partners[b.id]]


# --------------------------------------------------------------------------- coloring
# proj/src/coloring.cpp

@dataclass
class ConstraintSet:
    payload: tuple   # ((box, tag), ...) sorted
    zero: tuple      # sorted
    owners: list


def build_constraints(tree, adj, level, mode):
    """proj/src/coloring.cpp:55-113 (kH1, kUnifStage1, kUnifStage2, kLeaf)."""
    index = {}
    sets = []

    def add(payload, zero, owner):
        key = (payload, zero)
        if key in index:
            sets[index[key]].owners.append(owner)
        else:
            index[key] = len(sets)
            sets.append(ConstraintSet(payload, zero, [owner]))

    if mode == H1:
        for a, b in admissible_pairs(tree, adj, level):
            z = set(adj.neighbors[a]) | set(adj.interaction[a]) | set(adj.coarse_leaf_neighbors[a])
            z.discard(b)
            add(((b, GAUSSIAN),), tuple(sorted(z)), (a, b))
    elif mode == UNIF2:
        # adjoint-side probe carrying the alpha basis, observed at I_beta
        for a, b in admissible_pairs(tree, adj, level):
            z = set(adj.neighbors[b]) | set(adj.interaction[b]) | set(adj.coarse_leaf_neighbors[b])
            z.discard(a)
            add(((a, BASIS),), tuple(sorted(z)), (a, b))
    elif mode == UNIF1:
        if level < 2 or level > tree.depth:
            raise ValueError("sampling level out of range")
        for a in tree.level_boxes(level):
            if not adj.interaction[a]:
                continue
            payload = tuple((b, GAUSSIAN) for b in adj.interaction[a])
            z = sorted(set(adj.neighbors[a]) | set(adj.coarse_leaf_neighbors[a]))
            add(payload, tuple(z), (a, -1))
    elif mode == LEAF:
        for lam, mu in dense_pairs(tree, adj):
            z = [x for x in adj.dense_partners[lam] if x != mu]
            add(((mu, IDENTITY),), tuple(z), (lam, mu))
    else:
        raise ValueError("unsupported mode")
    return sets


def incompatible(a: ConstraintSet, b: ConstraintSet) -> bool:
    """proj/src/coloring.cpp:115-146."""
    za, zb = set(a.zero), set(b.zero)
    if any(p in zb for p, _ in a.payload) or any(p in za for p, _ in b.payload):
        return True
    tb = dict(b.payload)
    return any(p in tb and tb[p] != t for p, t in a.payload)


def build_graph(sets):
    """proj/src/coloring.cpp:154-167: the pairwise `incompatible` scan,
    vectorized with incidence matrices for up to 6000 sets and enumerated per
    box above that (same edge set; build_graph_literal is the scan as
    written, tests/test_oracle.py pins all three against each other)."""
    n = len(sets)
    if 0 < n <= 6000:
        # the same pairwise predicate, evaluated for all (i, j) at once with
        # incidence matrices: payload-hits-zero either way, or one box with
        # two different payload tags
        nb = 1 + max(max([b for s in sets for b, _ in s.payload] + [0]),
                     max([z for s in sets for z in s.zero] + [0]))
        P = np.zeros((n, nb), dtype=np.float32)
        Z = np.zeros((n, nb), dtype=np.float32)
        T = [np.zeros((n, nb), dtype=np.float32) for _ in range(3)]
        for i, s in enumerate(sets):
            for b, t in s.payload:
                P[i, b] = 1.0
                T[t][i, b] = 1.0
            for z in s.zero:
                Z[i, z] = 1.0
        hit = (P @ Z.T) > 0
        inc = hit | hit.T
        for a in range(3):
            for b in range(3):
                if a != b:
                    inc |= (T[a] @ T[b].T) > 0
        np.fill_diagonal(inc, False)
        return [list(np.nonzero(inc[i])[0].astype(int)) for i in range(n)]
    return _build_graph_indexed(sets)


def build_graph_literal(sets):
    """proj/src/coloring.cpp:154-167 as written: every pair (i < j) through
    `incompatible` (O(V^2); small inputs, to pin the faster forms)."""
    n = len(sets)
    edges = [[] for _ in range(n)]
    for i in range(n):
        for j in range(i + 1, n):
            if incompatible(sets[i], sets[j]):
                edges[i].append(j)
                edges[j].append(i)
    return edges


def _build_graph_indexed(sets, chunk=1 << 24):
    """The same edge set as the pairwise scan, enumerated per box: sets whose
    payload holds box b clash with every set whose zero set holds b, and with
    each other when their tags for b differ (`incompatible`'s three clauses).
    Candidate pairs are encoded as i * n + j and de-duplicated with numpy."""
    n = len(sets)
    pay, zer = {}, {}
    for i, s in enumerate(sets):
        for b, t in s.payload:
            pay.setdefault(b, []).append((i, t))
        for z in s.zero:
            zer.setdefault(z, []).append(i)
    parts, pending, found = [], [], 0

    def flush():
        nonlocal pending, found
        if pending:
            parts.append(np.unique(np.concatenate(pending)))
            pending, found = [], 0

    for b, lst in pay.items():
        pi = np.array([i for i, _ in lst], dtype=np.int64)
        zs = zer.get(b)
        if zs:
            zi = np.array(zs, dtype=np.int64)
            codes = (pi[:, None] * n + zi[None, :]).ravel()
            pending += [codes, (zi[:, None] * n + pi[None, :]).ravel()]
            found += 2 * codes.size
        tags = np.array([t for _, t in lst])
        if len(lst) > 1 and np.any(tags != tags[0]):
            ii, jj = np.nonzero(tags[:, None] != tags[None, :])
            pending.append(pi[ii] * n + pi[jj])
            found += ii.size
        if found > chunk:
            flush()
    flush()
    if not parts:
        return [[] for _ in range(n)]
    codes = np.unique(np.concatenate(parts))
    i, j = codes // n, codes % n
    keep = i != j
    i, j = i[keep], j[keep]
    # codes are sorted by (i, j): split into per-vertex sorted lists
    starts = np.searchsorted(i, np.arange(n + 1))
    jl = j.tolist()
    return [jl[starts[v]:starts[v + 1]] for v in range(n)]


def dsatur_color(edges):
    """proj/src/coloring.cpp:169-216: max (saturation, uncolored degree, -v);
    smallest free color. Returns (colors, num_colors)."""
    import heapq
    n = len(edges)
    color = [-1] * n
    if n == 0:
        return color, 0
    if n <= 20000:
        # same rule by direct arg-max over the uncolored vertices: key
        # (saturation, uncolored degree, -v), ties impossible
        col = np.full(n, -1, dtype=np.int64)
        seen = np.zeros((n, 64), dtype=bool)
        sat = np.zeros(n, dtype=np.int64)
        udeg = np.array([len(e) for e in edges], dtype=np.int64)
        adj = [np.asarray(e, dtype=np.int64) for e in edges]
        ncol = 0
        bits = np.int64(1) << 20  # > n and > any degree: lexicographic key
        order = bits - 1 - np.arange(n, dtype=np.int64)
        for _ in range(n):
            key = np.where(col < 0, (sat * bits + udeg) * bits + order, -1)
            v = int(np.argmax(key))
            used = seen[v]
            c = int(np.argmin(used)) if not used.all() else used.size
            if c >= seen.shape[1]:
                seen = np.concatenate([seen, np.zeros((n, seen.shape[1]), dtype=bool)], axis=1)
            col[v] = c
            ncol = max(ncol, c + 1)
            nb = adj[v]
            nb = nb[col[nb] < 0]
            udeg[nb] -= 1
            fresh = nb[~seen[nb, c]]
            seen[fresh, c] = True
            sat[fresh] += 1
        return [int(x) for x in col], ncol
    seen = [set() for _ in range(n)]
    udeg = [len(e) for e in edges]
    stamp = [0] * n
    heap = [(0, -udeg[v], v, 0) for v in range(n)]  # min-heap on (-sat, -udeg, v)
    heapq.heapify(heap)
    ncol = 0
    done = 0
    while done < n:
        negsat, negud, v, st = heapq.heappop(heap)
        if color[v] != -1 or st != stamp[v]:
            continue
        c = 0
        while c in seen[v]:
            c += 1
        color[v] = c
        ncol = max(ncol, c + 1)
        done += 1
        for w in edges[v]:
            if color[w] != -1:
                continue
            udeg[w] -= 1
            seen[w].add(c)
            stamp[w] += 1
            heapq.heappush(heap, (-len(seen[w]), -udeg[w], w, stamp[w]))
    return color, ncol


def plan_coloring(tree, sets, edges, mode):
    """proj/src/coloring.cpp:218-250."""
    color, ncol = dsatur_color(edges)
    if mode == UNIF2 or not tree.is_fully_populated():
        return color, ncol
    mod = {H1: 6, UNIF1: 5, LEAF: 3}[mode]
    relabel = {}
    tile = []
    for s in sets:
        box = s.owners[0][0] if mode == UNIF1 else s.payload[0][0]
        idx, mul = 0, 1
        for c in tree.box(box).coord:
            idx += (c % mod) * mul
            mul *= mod
        if idx not in relabel:
            relabel[idx] = len(relabel)
        tile.append(relabel[idx])
    if len(relabel) < ncol:
        return tile, len(relabel)
    return color, ncol


def payload_gaussian(tree, box, width, seed, level, phase):
    """proj/src/coloring.cpp:252-259."""
    return gaussian_matrix(len(tree.box(box).points), width, mix_seed(seed, level, box, phase))


@dataclass
class BlockTestMatrix:
    rows: int
    width: int
    seed: int
    level: int
    phase: int
    payload: list
    zero: list
    serves: list

    def realize(self, tree, basis_table=None):
        """proj/src/coloring.cpp:261-291."""
        out = np.zeros((self.rows, self.width))
        for box, tag in self.payload:
            pts = tree.box(box).points
            if tag == GAUSSIAN:
                blk = payload_gaussian(tree, box, self.width, self.seed, self.level, self.phase)
            elif tag == BASIS:
                if basis_table is None or box not in basis_table:
                    raise RuntimeError("missing basis for payload box")
                basis = basis_table[box]
                blk = np.zeros((len(pts), self.width))
                blk[:, :basis.shape[1]] = basis
            else:
                blk = np.zeros((len(pts), self.width))
                k = min(len(pts), self.width)
                blk[np.arange(k), np.arange(k)] = 1.0
            out[pts, :] = blk
        return out


def assemble_test_matrices(sets, color, ncol, tree, level, width, seed, phase, basis_table=None):
    """proj/src/coloring.cpp:293-332 (basis payloads: width = the widest
    basis of the color)."""
    mats = [BlockTestMatrix(tree.num_points, width, seed, level, phase, [], [], []) for _ in range(ncol)]
    merged = [dict() for _ in range(ncol)]
    zeros = [set() for _ in range(ncol)]
    for i, s in enumerate(sets):
        c = color[i]
        mats[c].serves.append(i)
        for box, tag in s.payload:
            if box in merged[c] and merged[c][box] != tag:
                raise AssertionError("conflicting payload tags within a color")
            merged[c][box] = tag
        zeros[c].update(s.zero)
    for c in range(ncol):
        mats[c].payload = sorted(merged[c].items())
        mats[c].zero = sorted(zeros[c])
        bases = [b for b, t in mats[c].payload if t == BASIS]
        if bases:
            if basis_table is None or any(b not in basis_table for b in bases):
                raise RuntimeError("missing basis for payload box")
            mats[c].width = max([1] + [basis_table[b].shape[1] for b in bases])
    return mats


@dataclass
class Plan:
    sets: list
    edges: list
    color: list
    matrices: list
    block_to_matrix: dict
    box_to_matrix: dict = field(default_factory=dict)


def pattern_index(box, mod):
    """proj/src/peeling.cpp:88-96."""
    idx, mul = 0, 1
    for c in box.coord:
        idx += (c % mod) * mul
        mul *= mod
    return idx


def fallback_pattern_matrices(tree, adj, level, mode, width, seed, phase):
    """proj/src/coloring.cpp:334-407: the 6^d / 5^d / 3^d shifted grid
    patterns of a fully populated uniform tree (no graph, no coloring)."""
    if not tree.is_fully_populated():
        raise ValueError("pattern test matrices require a fully populated uniform tree")
    if mode == UNIF2:
        raise ValueError("no pattern construction for basis probes")
    d = tree.dim
    mod = 6 if mode == H1 else 5 if mode == UNIF1 else 3
    if mode == LEAF:
        level = tree.depth
    if level < 2 or level > tree.depth:
        raise ValueError("sampling level out of range")
    mats = []
    for idx in range(mod ** d):
        shift, rem = [], idx
        for _ in range(d):
            shift.append(rem % mod)
            rem //= mod
        m = BlockTestMatrix(tree.num_points, width, seed, level, phase, [], [], [])
        for b in tree.level_boxes(level):
            coord = tree.box(b).coord
            if mode == UNIF1:
                # zero on the 3^d cluster around each aligned center, payload elsewhere
                active = not all((coord[j] - shift[j]) % mod in (0, 1, mod - 1) for j in range(d))
            else:
                active = all(coord[j] % mod == shift[j] for j in range(d))
            if active:
                m.payload.append((b, IDENTITY if mode == LEAF else GAUSSIAN))
            else:
                m.zero.append(b)
        mats.append(m)
    return mats


def make_plan(tree, adj, level, mode, width, seed, phase, basis_table=None, strategy="graph"):
    """proj/src/peeling.cpp:98-154 (graph strategy; the fallback-pattern
    strategy for every mode but the basis probes, :131-153)."""
    if strategy != "graph" and mode != UNIF2:
        mats = fallback_pattern_matrices(tree, adj, level, mode, width, seed, phase)
        mod = 6 if mode == H1 else 5 if mode == UNIF1 else 3
        b2m, box2m = {}, {}
        if mode == H1:
            for a, b in admissible_pairs(tree, adj, level):
                b2m[(a, b)] = pattern_index(tree.box(b), mod)
        elif mode == UNIF1:
            for a in tree.level_boxes(level):
                if adj.interaction[a]:
                    box2m[a] = pattern_index(tree.box(a), mod)
        else:
            for lam, mu in dense_pairs(tree, adj):
                b2m[(lam, mu)] = pattern_index(tree.box(mu), mod)
        return Plan([], [], [], mats, b2m, box2m)
    sets = build_constraints(tree, adj, level, mode)
    if not sets:
        return Plan([], [], [], [], {})
    edges = build_graph(sets)
    color, ncol = plan_coloring(tree, sets, edges, mode)
    mats = assemble_test_matrices(sets, color, ncol, tree, level, width, seed, phase, basis_table)
    b2m, box2m = {}, {}
    for i, s in enumerate(sets):
        for o in s.owners:
            if mode == UNIF1:
                box2m[o[0]] = color[i]
            else:
                b2m[o] = color[i]
    return Plan(sets, edges, color, mats, b2m, box2m)


# --------------------------------------------------------------------------- linalg
# proj/src/linalg.cpp

QR_RANK_DROP_TOL = 1e-14   # proj/include/hpeel/linalg.hpp:33
PINV_CUTOFF = 1e-12        # proj/include/hpeel/linalg.hpp:35


def qr_orthonormal(m, max_rank=-1):
    """proj/src/linalg.cpp:53-78: column-pivoted Householder QR (LAPACK
    dgeqp3 standing in for Eigen::ColPivHouseholderQR), keep the leading
    columns with |R_jj| > 1e-14 |R_00|, capped at max_rank."""
    m = np.asarray(m, dtype=np.float64)
    if m.shape[0] == 0 or m.shape[1] == 0:
        return np.zeros((m.shape[0], 0))
    if not np.all(np.isfinite(m)):
        raise ValueError("non-finite matrix in qr")
    q, r, _ = scipy.linalg.qr(m, mode="economic", pivoting=True)
    kmax = min(m.shape)
    p0 = abs(r[0, 0])
    keep = 0
    while keep < kmax and abs(r[keep, keep]) > QR_RANK_DROP_TOL * p0:
        keep += 1
    if max_rank >= 0:
        keep = min(keep, max_rank)
    return q[:, :keep]


def svd_trunc_fixed(m, k):
    """svd_trunc for TruncationSpec::fixed_rank (proj/src/linalg.cpp:80-108):
    the leading min(k, #{sigma > 0}) left singular vectors (LAPACK dgesdd for
    Eigen's BDCSVD: signs of the vectors are not pinned)."""
    if m.shape[0] == 0 or m.shape[1] == 0:
        return np.zeros((m.shape[0], 0))
    if not np.isfinite(m).all():
        raise ValueError("non-finite matrix in svd")
    u, sv, _ = scipy.linalg.svd(m, full_matrices=False, lapack_driver="gesdd")
    keep = 0
    while keep < min(len(sv), k) and sv[keep] > 0.0:
        keep += 1
    return u[:, :keep]


def pinv_apply(c, rhs):
    """proj/src/linalg.cpp:110-127 (SVD cutoff 1e-12 sigma_1)."""
    c = np.asarray(c, dtype=np.float64)
    if c.shape[0] != rhs.shape[0]:
        raise ValueError("pinv_apply: row mismatch")
    if c.shape[0] == 0 or c.shape[1] == 0:
        return np.zeros((c.shape[1], rhs.shape[1]))
    u, s, vt = np.linalg.svd(c, full_matrices=False)
    inv = np.where(s > PINV_CUTOFF * s[0], 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return vt.T @ (inv[:, None] * (u.T @ rhs))


# --------------------------------------------------------------------------- operators

def kernel_matrix(kind, xi, xj, same=None, param=0.1):
    """Kernel blocks of the BASELINE.json on-the-fly operators, evaluated on
    raw coordinates: log|x-y| (A_ii = 0), 1/(4 pi |x-y|) (A_ii = 0),
    exp(-|x-y|/param)."""
    diff = xi[:, None, :] - xj[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    with np.errstate(divide="ignore"):
        if kind == "log":
            k = np.log(r)
        elif kind == "invdist4pi":
            k = 1.0 / (4.0 * math.pi * r)
        elif kind == "exp":
            return np.exp(-r / param)
        else:
            raise ValueError(kind)
    if same is not None:
        k[same] = 0.0
    return k


def _nonzero_rows(x):
    return np.nonzero(np.any(x != 0.0, axis=1))[0]


class DenseOperator:
    """proj/include/hpeel/operators.hpp:56-69."""

    def __init__(self, a):
        self.a = np.asarray(a, dtype=np.float64)
        self.shape = self.a.shape

    def apply(self, x):
        return self.a @ x

    def apply_adjoint(self, x):
        return self.a.T @ x

    def apply_rows(self, x, rows, adjoint=False):
        """(A x)[rows] (or (A^T x)[rows]) over the nonzero rows of x only."""
        nz = _nonzero_rows(x)
        a = self.a.T if adjoint else self.a
        return a[np.ix_(rows, nz)] @ x[nz]


class KernelOperator:
    """On-the-fly kernel black box (row-chunked K(X, X) @ x), for sizes where
    a dense A does not fit."""

    def __init__(self, kind, points, param=0.1, chunk=2048):
        self.kind = kind
        self.x = np.asarray(points, dtype=np.float64)
        if self.x.ndim == 1:
            self.x = self.x[:, None]
        self.param = param
        self.chunk = chunk
        n = self.x.shape[0]
        self.shape = (n, n)

    def block(self, i0, i1):
        n = self.shape[0]
        same = None
        if self.kind != "exp":
            same = (np.arange(i0, i1)[:, None] == np.arange(n)[None, :])
        return kernel_matrix(self.kind, self.x[i0:i1], self.x, same, self.param)

    def apply(self, x):
        n = self.shape[0]
        y = np.empty((n, x.shape[1]))
        for i0 in range(0, n, self.chunk):
            i1 = min(n, i0 + self.chunk)
            y[i0:i1] = self.block(i0, i1) @ x
        return y

    apply_adjoint = apply  # symmetric kernels

    def apply_rows(self, x, rows, adjoint=False):
        """(K x)[rows] over the nonzero rows of x only (K symmetric); row
        chunks on a thread pool (numpy releases the GIL in both steps)."""
        nz = _nonzero_rows(x)
        y = np.empty((len(rows), x.shape[1]))
        xn = x[nz]
        xz = self.x[nz]
        step = max(64, min(self.chunk, (1 << 22) // max(len(nz), 1)))

        def work(i0):
            r = rows[i0:i0 + step]
            same = (r[:, None] == nz[None, :]) if self.kind != "exp" else None
            y[i0:i0 + len(r)] = kernel_matrix(self.kind, self.x[r], xz, same, self.param) @ xn

        starts = list(range(0, len(rows), step))
        threads = getattr(self, "threads", os.cpu_count() or 1)
        if threads > 1 and len(starts) > 1:
            from concurrent.futures import ThreadPoolExecutor
            with _small_blas(), ThreadPoolExecutor(threads) as ex:
                list(ex.map(work, starts))
        else:
            for i0 in starts:
                work(i0)
        return y


# --------------------------------------------------------------------------- H1 rep
# proj/src/hmatrix.cpp:21-150

class H1Rep:
    def __init__(self, tree, adj):
        self.tree = tree
        self.adj = adj
        self.built_level = 1
        self.dense_ready = False
        self.levels = [dict() for _ in range(tree.depth + 1)]
        self.dense = {}

    def _check(self, level):
        if level > self.built_level:
            raise RuntimeError(f"h1 apply: representation incomplete for level {level}")

    def apply_truncated(self, level, x):
        """proj/src/hmatrix.cpp:86-100."""
        self._check(level)
        y = np.zeros_like(x)
        for l in range(2, min(level, self.tree.depth) + 1):
            for (a, b), (u, bb, v) in sorted(self.levels[l].items()):
                y[self.tree.box(a).points] += u @ (bb @ (v.T @ x[self.tree.box(b).points]))
        return y

    def apply_truncated_adjoint(self, level, x):
        """proj/src/hmatrix.cpp:102-116."""
        self._check(level)
        y = np.zeros_like(x)
        for l in range(2, min(level, self.tree.depth) + 1):
            for (a, b), (u, bb, v) in sorted(self.levels[l].items()):
                y[self.tree.box(b).points] += v @ (bb.T @ (u.T @ x[self.tree.box(a).points]))
        return y

    def _box_at_level(self, l):
        """point -> its box at level l (-1 if the point's leaf is coarser)."""
        cache = self.__dict__.setdefault("_bal", {})
        if l not in cache:
            m = np.full(self.tree.num_points, -1, dtype=np.int64)
            for b in self.tree.level_boxes(l):
                m[self.tree.box(b).points] = b
            cache[l] = m
        return cache[l]

    def apply_truncated_rows(self, level, x, mask, adjoint=False):
        """Rows `mask` of apply_truncated(_adjoint)(level, x): only the pairs
        whose column block of x is nonzero and whose row block meets the mask
        contribute there (the same sums, in the same sorted pair order,
        restricted to the rows the extraction reads)."""
        self._check(level)
        y = np.zeros_like(x)
        nz = _nonzero_rows(x)
        rows_all = np.nonzero(mask)[0]
        for l in range(2, min(level, self.tree.depth) + 1):
            bal = self._box_at_level(l)
            srcs = set(np.unique(bal[nz]).tolist()) - {-1}
            dsts = set(np.unique(bal[rows_all]).tolist()) - {-1}
            if not srcs or not dsts:
                continue
            for (a, b), (u, bb, v) in sorted(self.levels[l].items()):
                src, dst = (a, b) if adjoint else (b, a)
                if src not in srcs or dst not in dsts:
                    continue
                rows = self.tree.box(dst).points
                sel = mask[rows]
                xs = x[self.tree.box(src).points]
                if adjoint:
                    y[rows[sel]] += v[sel] @ (bb.T @ (u.T @ xs))
                else:
                    y[rows[sel]] += u[sel] @ (bb @ (v.T @ xs))
        return y

    def _dense(self, x, y, adjoint):
        """proj/src/hmatrix.cpp:59-73."""
        for (lam, mu), d in sorted(self.dense.items()):
            rows = self.tree.box(mu if adjoint else lam).points
            cols = self.tree.box(lam if adjoint else mu).points
            y[rows] += (d.T if adjoint else d) @ x[cols]

    def apply(self, x):
        if not self.dense_ready:
            raise RuntimeError("h1 apply: dense blocks missing")
        y = self.apply_truncated(self.tree.depth, x)
        self._dense(x, y, False)
        return y

    def apply_adjoint(self, x):
        if not self.dense_ready:
            raise RuntimeError("h1 apply: dense blocks missing")
        y = self.apply_truncated_adjoint(self.tree.depth, x)
        self._dense(x, y, True)
        return y

    def storage(self):
        """proj/src/hmatrix.cpp:132-150 (total scalars)."""
        t = 0
        for lv in self.levels:
            for u, b, v in lv.values():
                t += u.size + b.size + v.size
        t += sum(d.size for d in self.dense.values())
        return t


class UnifH1Rep:
    """Uniform H1 (proj/include/hpeel/hmatrix.hpp:73-97, proj/src/hmatrix.cpp:152-250):
    one row basis U_a and one column basis V_b per box, a coupling B_ab per
    admissible pair."""

    def __init__(self, tree, adj):
        self.tree = tree
        self.adj = adj
        self.built_level = 1
        self.dense_ready = False
        self.box_u = {}
        self.box_v = {}
        self.level_b = [dict() for _ in range(tree.depth + 1)]
        self.dense = {}

    def _check(self, level):
        if level > self.built_level:
            raise RuntimeError(f"unif-h1 apply: representation incomplete for level {level}")

    def apply_truncated(self, level, x):
        """proj/src/hmatrix.cpp:165-189."""
        self._check(level)
        y = np.zeros_like(x)
        for l in range(2, min(level, self.tree.depth) + 1):
            qhat, uhat = {}, {}
            for (a, b), bb in sorted(self.level_b[l].items()):
                if b not in qhat:
                    qhat[b] = self.box_v[b].T @ x[self.tree.box(b).points]
                uhat[a] = uhat.get(a, 0) + bb @ qhat[b]
            for a in sorted(uhat):
                y[self.tree.box(a).points] += self.box_u[a] @ uhat[a]
        return y

    def apply_truncated_adjoint(self, level, x):
        """proj/src/hmatrix.cpp:191-215."""
        self._check(level)
        y = np.zeros_like(x)
        for l in range(2, min(level, self.tree.depth) + 1):
            qhat, vhat = {}, {}
            for (a, b), bb in sorted(self.level_b[l].items()):
                if a not in qhat:
                    qhat[a] = self.box_u[a].T @ x[self.tree.box(a).points]
                vhat[b] = vhat.get(b, 0) + bb.T @ qhat[a]
            for b in sorted(vhat):
                y[self.tree.box(b).points] += self.box_v[b] @ vhat[b]
        return y

    def apply_truncated_rows(self, level, x, mask, adjoint=False):
        out = self.apply_truncated_adjoint(level, x) if adjoint else self.apply_truncated(level, x)
        out[~mask] = 0.0
        return out

    _dense = H1Rep._dense
    apply = H1Rep.apply
    apply_adjoint = H1Rep.apply_adjoint

    def storage(self):
        t = sum(u.size for u in self.box_u.values()) + sum(v.size for v in self.box_v.values())
        t += sum(b.size for lv in self.level_b for b in lv.values())
        t += sum(d.size for d in self.dense.values())
        return t


# --------------------------------------------------------------------------- driver
# proj/src/peeling.cpp

class PhaseTimes(dict):
    """Wall seconds per phase of the oracle's compress (bench.py reference
    arm): plan, realize, apply (black box), peel (apply_truncated), qr, bsolve."""

    def add(self, key, t0):
        import time
        self[key] = self.get(key, 0.0) + (time.perf_counter() - t0)


def _pair_map(fn, pairs):
    """fn over the pairs in order; independent per-pair solves run on a
    thread pool when there are many (LAPACK releases the GIL; the results and
    their order are those of the serial loop, proj/src/peeling.cpp:245-270)."""
    threads = os.cpu_count() or 1
    if threads == 1 or len(pairs) < 256:
        return [fn(ab) for ab in pairs]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(fn, pairs, chunksize=64))


def _small_blas():
    """Per-pair QR / SVD / small GEMMs on one BLAS thread: a threaded BLAS is
    ~50x slower on 64 x 48 matrices (thread start-up per call), and the
    reference runs these serially anyway (proj/src/peeling.cpp:245-270)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except ImportError:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def _now():
    import time
    return time.perf_counter()


def _served_rows(tree, plan, m_index, owner_row=0):
    """Tree points of the row boxes of the pairs a color serves (the rows the
    extraction reads back from its sample; owner_row 1: the column box, for
    the uniform driver's adjoint basis probes)."""
    pts = [tree.box(o[owner_row]).points for i in plan.matrices[m_index].serves for o in plan.sets[i].owners]
    return np.unique(np.concatenate(pts)) if pts else np.zeros(0, dtype=np.int64)


def _residual_samples(op, rep, prev_level, plan, adjoint, phase=None, times=None, restrict=False, raw=None,
                      basis_table=None, owner_row=0):
    """proj/src/peeling.cpp:158-178. Returns (samples, cols). restrict=True
    computes only the rows the extraction reads (value-identical on those
    rows: the same products over the nonzero rows of Omega; other rows 0).
    `raw` (a list) receives each color's black-box product before peeling."""
    times = PhaseTimes() if times is None else times
    samples, cols = [], 0
    for ci, m in enumerate(plan.matrices):
        if not m.payload:
            samples.append(None)
            if raw is not None:
                raw.append(None)
            continue
        if phase is not None:
            m = BlockTestMatrix(m.rows, m.width, m.seed, m.level, phase, m.payload, m.zero, m.serves)
        t0 = _now()
        omega = m.realize(rep.tree, basis_table)
        times.add("realize", t0)
        cols += omega.shape[1]
        if restrict:
            rows = _served_rows(rep.tree, plan, ci, owner_row)
            mask = np.zeros(omega.shape[0], dtype=bool)
            mask[rows] = True
            t0 = _now()
            y = np.zeros_like(omega)
            y[rows] = op.apply_rows(omega, rows, adjoint)
            times.add("apply", t0)
            if raw is not None:
                raw.append(y.copy())
            if prev_level >= 2:
                t0 = _now()
                y[rows] -= rep.apply_truncated_rows(prev_level, omega, mask, adjoint)[rows]
                times.add("peel", t0)
            samples.append(y)
            continue
        t0 = _now()
        y = op.apply_adjoint(omega) if adjoint else op.apply(omega)
        times.add("apply", t0)
        if raw is not None:
            raw.append(y)
        if prev_level >= 2:
            t0 = _now()
            y = y - (rep.apply_truncated_adjoint(prev_level, omega) if adjoint
                     else rep.apply_truncated(prev_level, omega))
            times.add("peel", t0)
        samples.append(y)
    return samples, cols


def run_h1(op, tree, adj, k, p, seed, report, capture=None, times=None, restrict=False, raw_capture=None,
           strategy="graph"):
    """proj/src/peeling.cpp:211-275 (Alg. 4.1)."""
    times = PhaseTimes() if times is None else times
    rep = H1Rep(tree, adj)
    r = k + p
    for l in range(2, tree.depth + 1):
        pairs = admissible_pairs(tree, adj, l)
        if not pairs:
            continue
        ps = set(pairs)
        if any((b, a) not in ps for a, b in pairs):
            raise AssertionError("asymmetric admissibility structure")
        t0 = _now()
        plan = make_plan(tree, adj, l, H1, r, seed, 0, strategy=strategy)
        times.add("plan", t0)
        yraw, zraw = ([], []) if raw_capture is not None else (None, None)
        ys, fcols = _residual_samples(op, rep, l - 1, plan, False, times=times, restrict=restrict, raw=yraw)
        u_bases = {}
        t0 = _now()
        with _small_blas():
            qs = _pair_map(lambda ab: qr_orthonormal(ys[plan.block_to_matrix[ab]][tree.box(ab[0]).points], k),
                           pairs)
            for ab, q in zip(pairs, qs):
                u_bases[ab] = q
        times.add("qr", t0)
        zs, acols = _residual_samples(op, rep, l - 1, plan, True, phase=1, times=times, restrict=restrict, raw=zraw)
        if raw_capture is not None:
            raw_capture[l] = {(a, b): (yraw[plan.block_to_matrix[(a, b)]][tree.box(a).points],
                                       zraw[plan.block_to_matrix[(a, b)]][tree.box(a).points])
                              for a, b in pairs}
        if capture is not None:
            capture[l] = {(a, b): (ys[plan.block_to_matrix[(a, b)]][tree.box(a).points],
                                   zs[plan.block_to_matrix[(a, b)]][tree.box(a).points])
                          for a, b in pairs}
        def solve(ab):
            a, b = ab
            z = zs[plan.block_to_matrix[(b, a)]]
            u = u_bases[(a, b)]
            v = qr_orthonormal(z[tree.box(b).points], k)
            g = payload_gaussian(tree, b, r, seed, l, 0)
            gp = payload_gaussian(tree, a, r, seed, l, 1)
            yb = ys[plan.block_to_matrix[(a, b)]][tree.box(a).points]
            middle = gp.T @ yb
            left = pinv_apply(gp.T @ u, middle)
            bmat = pinv_apply((v.T @ g).T, left.T).T
            return (u, bmat, v)

        t0 = _now()
        with _small_blas():
            blocks = _pair_map(solve, pairs)
        times.add("bsolve", t0)  # the V QR included
        for ab, blk in zip(pairs, blocks):
            rep.levels[l][ab] = blk
        rep.built_level = l
        report.append({"phase": "h1", "level": l, "colors": len(plan.matrices),
                       "forward_cols": fcols, "adjoint_cols": acols})
    rep.built_level = tree.depth
    return rep


def run_uniform(op, tree, adj, k, p, seed, report, capture=None, times=None, restrict=False):
    """proj/src/peeling.cpp:291-454 for the uniform-H1 target (no nesting):
    stage 1 samples each box against its whole interaction list and takes the
    row basis U_a from them; stage 2 loads U_a into adjoint probes, reads
    S_ab = A_ab^T U_a at I_b, takes the column basis V_b from sum_a S_ab and
    the couplings B_ab = S_ab^T V_b. The bases are the leading left singular
    vectors (basis_from_sample with a sigma out-parameter takes the svd_trunc
    branch, peeling.cpp:63-71, :341, :406), not the pivoted-QR range finder of
    the H1 driver. No device path exists for this format."""
    times = PhaseTimes() if times is None else times
    rep = UnifH1Rep(tree, adj)
    r = k + p
    for l in range(2, tree.depth + 1):
        pairs = admissible_pairs(tree, adj, l)
        if not pairs:
            continue
        ps = set(pairs)
        if any((b, a) not in ps for a, b in pairs):
            raise AssertionError("asymmetric admissibility structure")
        # stage 1 (forward phase, Gaussian payloads on the interaction lists)
        plan1 = make_plan(tree, adj, l, UNIF1, r, seed, 0)
        ys, fcols = _residual_samples(op, rep, l - 1, plan1, False, times=times, restrict=restrict)
        for a in tree.level_boxes(l):
            if a not in plan1.box_to_matrix:
                continue
            sample = ys[plan1.box_to_matrix[a]][tree.box(a).points]
            with _small_blas():
                rep.box_u[a] = svd_trunc_fixed(sample, k)
        report.append({"phase": "unif-stage1", "level": l, "colors": len(plan1.matrices),
                       "forward_cols": fcols, "adjoint_cols": 0})
        # stage 2 (adjoint probes carrying the stage-1 bases)
        basis_table = {a: rep.box_u[a] for a in tree.level_boxes(l) if adj.interaction[a]}
        plan2 = make_plan(tree, adj, l, UNIF2, r, seed, 1, basis_table)
        zs, acols = _residual_samples(op, rep, l - 1, plan2, True, times=times, restrict=restrict,
                                      basis_table=basis_table, owner_row=1)
        projected = {}
        for a, b in pairs:
            z = zs[plan2.block_to_matrix[(a, b)]]
            projected[(a, b)] = z[tree.box(b).points][:, :rep.box_u[a].shape[1]]
        if capture is not None:
            capture[l] = {"u": {a: rep.box_u[a] for a in basis_table}, "s": dict(projected)}
        for b in tree.level_boxes(l):
            width = max([0] + [projected[(a, b)].shape[1] for a in adj.interaction[b]])
            if width == 0:
                continue
            acc = np.zeros((len(tree.box(b).points), width))
            for a in adj.interaction[b]:
                sab = projected[(a, b)]
                acc[:, :sab.shape[1]] += sab
            with _small_blas():
                rep.box_v[b] = svd_trunc_fixed(acc, k)
        for a, b in pairs:
            rep.level_b[l][(a, b)] = projected[(a, b)].T @ rep.box_v[b]
        rep.built_level = l
        report.append({"phase": "unif-stage2", "level": l, "colors": len(plan2.matrices),
                       "forward_cols": 0, "adjoint_cols": acols})
    rep.built_level = tree.depth
    return rep


def extract_leaf(op, rep, seed, report, capture=None, times=None, restrict=False, strategy="graph"):
    """proj/src/peeling.cpp:490-524."""
    times = PhaseTimes() if times is None else times
    tree, adj = rep.tree, rep.adj
    if rep.built_level < tree.depth:
        raise RuntimeError("leaf extraction needs all admissible levels built")
    width = tree.max_leaf_size()
    t0 = _now()
    plan = make_plan(tree, adj, tree.depth, LEAF, width, seed, 0, strategy=strategy)
    times.add("leaf_plan", t0)
    leaf_times = PhaseTimes()
    ys, fcols = _residual_samples(op, rep, tree.depth, plan, False, times=leaf_times, restrict=restrict)
    for key, v in leaf_times.items():
        times["leaf_" + key] = times.get("leaf_" + key, 0.0) + v
    for lam, mu in dense_pairs(tree, adj):
        y = ys[plan.block_to_matrix[(lam, mu)]]
        blk = y[tree.box(lam).points]
        if capture is not None:
            capture[(lam, mu)] = blk
        rep.dense[(lam, mu)] = blk[:, :len(tree.box(mu).points)]
    rep.dense_ready = True
    report.append({"phase": "leaf", "level": tree.depth, "colors": len(plan.matrices),
                   "forward_cols": fcols, "adjoint_cols": 0})


def compress(op, tree, k, p, seed, capture=None, leaf_capture=None, times=None, restrict=False, raw_capture=None,
             fmt="h1", strategy="graph"):
    """proj/src/peeling.cpp:576-639 for format h1. Returns (rep, report).
    `times` (a PhaseTimes) collects wall seconds per phase. restrict=True
    evaluates each color's black-box product and peeling only on the rows the
    extraction reads and over Omega's nonzero rows (row-restricted oracle for
    large N; the extracted samples are the same sums)."""
    if op.shape[0] != tree.num_points or op.shape[1] != tree.num_points:
        raise ValueError("operator and tree dimensions differ")
    if k < 1:
        raise ValueError("fixed rank must be >= 1")
    if p < 0:
        raise ValueError("negative oversampling")
    t0 = _now()
    adj = adjacency(tree)
    if times is not None:
        times.add("adjacency", t0)
    report = []
    if fmt == "unif-h1":
        rep = run_uniform(op, tree, adj, k, p, seed, report, capture, times, restrict)
    elif fmt == "h1":
        rep = run_h1(op, tree, adj, k, p, seed, report, capture, times, restrict, raw_capture, strategy)
    else:
        raise ValueError("unsupported format: " + fmt)
    extract_leaf(op, rep, seed, report, leaf_capture, times, restrict, strategy)
    return rep, report


def _power_norm_diff(a, b, iters, seed, n):
    """proj/src/linalg.cpp:179-196."""
    x = gaussian_matrix(n, 1, seed)
    x = x / np.linalg.norm(x)
    est = 0.0
    for _ in range(iters):
        y = a.apply(x)
        if b is not None:
            y = y - b.apply(x)
        z = a.apply_adjoint(y)
        if b is not None:
            z = z - b.apply_adjoint(y)
        nz = np.linalg.norm(z)
        if nz == 0.0:
            return 0.0
        est = math.sqrt(nz)
        x = z / nz
    return est


def rel_error_power_method(approx, ref, iters, seed):
    """proj/src/linalg.cpp:206-218."""
    n = ref.shape[0]
    err = _power_norm_diff(approx, ref, iters, mix_seed(seed, 11), n)
    base = _power_norm_diff(ref, None, iters, mix_seed(seed, 12), n)
    if base == 0.0:
        return 0.0 if err == 0.0 else math.inf
    return err / base


def _orth_gaussian(rows, cols, seed):
    """proj/src/operators.cpp:368-371: orthonormal basis of a Gaussian block."""
    return qr_orthonormal(gaussian_matrix(rows, cols, seed))


def synth_rank_structured(tree, adj, k, seed, fmt="h1"):
    """proj/src/operators.cpp:375-448 (H1 and uniform-H1 formats): per-pair
    rank-k blocks (H1: independent Gaussian factors; uniform: shared
    orthonormal bases per box with a Gaussian core) and Gaussian dense leaf
    blocks."""
    n = tree.num_points
    if n > 4096:
        raise ValueError("synthetic dense capped at 4096")
    a = np.zeros((n, n))
    bu, bv = {}, {}
    if fmt == "unif-h1":
        for l in range(tree.depth, 0, -1):
            for b in tree.level_boxes(l):
                rows = len(tree.box(b).points)
                bu[b] = _orth_gaussian(rows, k, mix_seed(seed, 101, b))
                bv[b] = _orth_gaussian(rows, k, mix_seed(seed, 102, b))
    elif fmt != "h1":
        raise ValueError("unsupported synthetic format: " + fmt)
    for l in range(2, tree.depth + 1):
        for al, be in admissible_pairs(tree, adj, l):
            rows, cols = tree.box(al).points, tree.box(be).points
            if fmt == "h1":
                gu = gaussian_matrix(len(rows), k, mix_seed(seed, 201, al, be))
                gv = gaussian_matrix(k, len(cols), mix_seed(seed, 202, al, be))
                a[np.ix_(rows, cols)] = gu @ gv / math.sqrt(k)
            else:
                core = gaussian_matrix(bu[al].shape[1], bv[be].shape[1], mix_seed(seed, 203, al, be))
                a[np.ix_(rows, cols)] = bu[al] @ core @ bv[be].T
    for lam, mu in dense_pairs(tree, adj):
        rows, cols = tree.box(lam).points, tree.box(mu).points
        a[np.ix_(rows, cols)] = gaussian_matrix(len(rows), len(cols), mix_seed(seed, 204, lam, mu))
    return a


# ---------------------------------------------------------------- .hrep files
# proj/src/serialize.cpp:14-270 (H1 format), little-endian; used by tests to
# check the device writer/reader byte for byte.
import struct as _struct

REP_MAGIC = 0x3150524C45455048     # "HPEELRP1", serialize.cpp:12
DENSE_MAGIC = 0x314D444C45455048   # "HPEELDM1", serialize.cpp:13
FORMAT_H1 = 1                      # RepFormat::kH1, hmatrix.hpp:16


def _put_matrix(out, m):
    """Writer::put_matrix, serialize.cpp:31-36 (rows, cols, column-major)."""
    m = np.asarray(m, dtype=np.float64)
    out.append(_struct.pack("<qq", m.shape[0], m.shape[1]))
    out.append(np.asfortranarray(m).tobytes(order="F"))


def save_rep_bytes(rep, k, leaf_capacity):
    """save_rep (serialize.cpp:156-188) for an oracle H1Rep: write_meta
    (:128-138), write_tree (:97-109), per level 0..depth the std::map-ordered
    blocks, then the dense blocks."""
    tree = rep.tree
    out = [_struct.pack("<Q", REP_MAGIC),
           _struct.pack("<Bqiiiiib", FORMAT_H1, tree.num_points, tree.dim, tree.depth, leaf_capacity, k,
                        rep.built_level, 1 if rep.dense_ready else 0)]
    out.append(_struct.pack("<iiqi", tree.dim, tree.leaf_capacity, tree.num_points, len(tree.boxes)))
    for b in tree.boxes:
        out.append(_struct.pack("<ii", b.level, b.parent))
        out.append(_struct.pack("<%dq" % tree.dim, *b.coord))
        out.append(_struct.pack("<i", len(b.children)) + _struct.pack("<%di" % len(b.children), *b.children))
        pts = [int(p) for p in b.points]
        out.append(_struct.pack("<i", len(pts)) + _struct.pack("<%di" % len(pts), *pts))
    for level in rep.levels:
        out.append(_struct.pack("<i", len(level)))
        for (a, b), (u, bb, v) in sorted(level.items()):
            out.append(_struct.pack("<ii", a, b))
            _put_matrix(out, u)
            _put_matrix(out, bb)
            _put_matrix(out, v)
    dense = rep.dense if rep.dense_ready else {}
    out.append(_struct.pack("<i", len(dense)))
    for (lam, mu), d in sorted(dense.items()):
        out.append(_struct.pack("<ii", lam, mu))
        _put_matrix(out, d)
    return b"".join(out)


class _Reader:
    def __init__(self, data):
        self.data, self.pos = data, 0

    def get(self, fmt):
        v = _struct.unpack_from("<" + fmt, self.data, self.pos)
        self.pos += _struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    def ints(self):
        n = self.get("i")
        return list(self.get("%di" % n)) if n > 1 else ([self.get("i")] if n == 1 else [])

    def matrix(self):
        r, c = self.get("qq")
        a = np.frombuffer(self.data, dtype="<f8", count=r * c, offset=self.pos).reshape((r, c), order="F")
        self.pos += 8 * r * c
        return np.array(a)


def load_rep_bytes(data):
    """load_rep (serialize.cpp:190-218) for the H1 format: returns
    (meta dict, boxes [(level, parent, coord, children, points)], levels
    [{(a, b): (u, b, v)}], dense {(lam, mu): d})."""
    r = _Reader(data)
    if r.get("Q") != REP_MAGIC:
        raise RuntimeError("not a representation file")
    fmt, n, dim, depth, leaf, rank, built, dense_ready = r.get("Bqiiiiib")
    meta = dict(format=fmt, n=n, dim=dim, depth=depth, leaf_capacity=leaf, rank=rank, built_level=built,
                dense_ready=bool(dense_ready))
    tdim, tleaf, tn, nboxes = r.get("iiqi")
    boxes = []
    for _ in range(nboxes):
        level, parent = r.get("ii")
        coord = r.get("%dq" % tdim)
        coord = (coord,) if tdim == 1 else tuple(coord)
        children = r.ints()
        points = r.ints()
        boxes.append((level, parent, coord, children, points))
    if fmt != FORMAT_H1:
        raise ValueError("only the H1 format is restated")
    levels = []
    for _ in range(depth + 1):
        cnt = r.get("i")
        lv = {}
        for _ in range(cnt):
            a, b = r.get("ii")
            lv[(a, b)] = (r.matrix(), r.matrix(), r.matrix())
        levels.append(lv)
    dense = {}
    for _ in range(r.get("i")):
        lam, mu = r.get("ii")
        dense[(lam, mu)] = r.matrix()
    if r.pos != len(data):
        raise RuntimeError("trailing bytes in representation file")
    return meta, boxes, levels, dense


def save_dense_matrix_bytes(m):
    """save_dense_matrix, serialize.cpp:252-256."""
    out = [_struct.pack("<Q", DENSE_MAGIC)]
    _put_matrix(out, m)
    return b"".join(out)
