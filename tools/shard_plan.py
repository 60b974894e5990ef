"""Per-rank device memory plan of the owner-computes sharded compress
(hp_shard_memory_plan) for a BASELINE config at full size, host only."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = configs.scaled(name, n) if n else configs.CONFIGS[name]
t0 = time.time()
tree = hp.build_tree(w.points(), w.leaf)
t1 = time.time()
plan = hp.shard_memory_plan(tree, w.rank, w.oversample, world)
one = hp.shard_memory_plan(tree, w.rank, w.oversample, 1)[0]
owner, cut, bounds = hp.shard_owners(tree, world)
gb = 1e9
print(json.dumps({
    "config": w.name, "n": w.n, "world": world, "depth": tree.depth, "cut_level": cut,
    "points_per_rank": [int(b - a) for a, b in zip(bounds[:-1], bounds[1:])],
    "per_rank_gb": [{"factors": round(r[0] / gb, 2), "dense": round(r[1] / gb, 2),
                     "level_max": round(r[2] / gb, 2), "total": round(r[3] / gb, 2)} for r in plan],
    "max_rank_total_gb": round(float(plan[:, 3].max()) / gb, 2),
    "single_gpu_gb": {"factors": round(one[0] / gb, 2), "dense": round(one[1] / gb, 2),
                      "level_max": round(one[2] / gb, 2), "total": round(one[3] / gb, 2)},
    "tree_s": round(t1 - t0, 1), "plan_s": round(time.time() - t1, 1)}, indent=1))
