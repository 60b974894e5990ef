"""Multi-rank host logic on CPU (gloo, world_size 2): every rank computes the
same work partition of every level's pairs and leaf blocks, the ranges tile
the index space exactly once, and the per-rank work is balanced; each rank
derives the same box ownership on its own, and the crossing-pair exchanges
it plans (what it sends to / expects from every peer, per level and phase)
match its peers' plans exactly. The device side of the same split is checked
on one GPU by emulation (tests/test_gpu_shard.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_03406_b200 import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _level_work(hp, tree, r, seed):
    out = []
    for l in range(2, tree.depth + 1):
        pairs = tree.admissible_pairs(l)
        if not pairs:
            continue
        plan = hp.plan(tree, l, "h1", r, seed, 0)
        b2m = plan.block_to_matrix()
        nnz = [sum(len(tree.box_points(b)) for b in plan.color_payload[c]) for c in range(plan.n_colors)]
        out.append([len(tree.box_points(a)) * nnz[b2m[(a, b)]] for a, b in pairs])
    return out


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2205_03406_b200 as hp
    w = configs.scaled("c3", 16384)
    tree = hp.build_tree(w.points(), w.leaf)
    works = _level_work(hp, tree, w.rank + w.oversample, 7)
    bounds = [hp.partition_ranges(wk, world) for wk in works]
    gathered = [None] * world
    dist.all_gather_object(gathered, bounds)
    if rank == 0:
        result["bounds"] = gathered
        result["works"] = works
    dist.barrier()
    dist.destroy_process_group()


def test_partition_is_identical_and_tiles_every_level():
    world = 2
    with mp.Manager() as mgr:
        result = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
        bounds, works = result["bounds"], result["works"]
    assert bounds[0] == bounds[1]
    for b, wk in zip(bounds[0], works):
        n = len(wk)
        assert b[0] == 0 and b[-1] == n and all(b[i] <= b[i + 1] for i in range(world))
        per_rank = [sum(wk[b[i]:b[i + 1]]) for i in range(world)]
        # contiguous ranges of pair work: each rank within one item of the ideal share
        ideal = sum(wk) / world
        assert max(per_rank) <= ideal + max(wk) + 1e-9


def test_partition_edge_cases(hp):
    assert hp.partition_ranges([], 3) == [0, 0, 0, 0]
    assert hp.partition_ranges([5.0], 4)[-1] == 1
    b = hp.partition_ranges(np.ones(1000), 8)
    assert [b[i + 1] - b[i] for i in range(8)] == [125] * 8
    b = hp.partition_ranges([1, 1, 1, 1, 10, 1, 1, 1], 2)
    assert b == [0, 4, 8]
    with pytest.raises(ValueError):
        hp.partition_ranges([1.0], 0)


def _exchange_worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2205_03406_b200 as hp
    out = {}
    for name, n in (("c3", 16384), ("c4", 16384), ("c2", 8192)):
        w = configs.scaled(name, n)
        tree = hp.build_tree(w.points(), w.leaf)
        owner, cut, bounds = hp.shard_owners(tree, world)
        plans = {}
        for level in range(2, tree.depth + 1):
            for phase in (1, 2):
                send, recv = hp.shard_exchange_counts(tree, w.rank, world, rank, level, phase)
                plans[(level, phase)] = (send.tolist(), recv.tolist())
        gathered = [None] * world
        dist.all_gather_object(gathered, (owner.tolist(), cut, bounds.tolist(), plans))
        out[name] = gathered
    if rank == 0:
        result["plans"] = out
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_plans_agree_across_ranks(world):
    with mp.Manager() as mgr:
        result = mgr.dict()
        mp.spawn(_exchange_worker, args=(world, _free_port(), result), nprocs=world, join=True)
        plans = dict(result["plans"])
    for name, per_rank in plans.items():
        owners = [p[0] for p in per_rank]
        assert all(o == owners[0] for o in owners), name
        assert all(p[1] == per_rank[0][1] and p[2] == per_rank[0][2] for p in per_rank), name
        moved = 0
        for key in per_rank[0][3]:
            for i in range(world):
                send_i = per_rank[i][3][key][0]
                for j in range(world):
                    recv_j = per_rank[j][3][key][1]
                    assert send_i[j] == recv_j[i], (name, key, i, j)
                    moved += send_i[j]
                assert send_i[i] == 0
        assert moved > 0, name  # some pairs cross the cut at every size tested
