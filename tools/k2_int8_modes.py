"""int8 K2 probe: full / no-MMA / no-evaluation apply times on one config."""
import sys
sys.path.insert(0, ".")
import paper_2205_03406_b200 as hp  # noqa: E402
from paper_2205_03406_b200 import configs  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = configs.CONFIGS[name] if len(sys.argv) < 3 else configs.scaled(name, int(sys.argv[2]))
pts = w.points()
t = hp.build_tree(pts, w.leaf)
op = hp.kernel_operator(w.kernel, pts, w.param)
for path in ("int8", "int8", "int8-nomma", "int8-noeval", "int8-nodsmem", "int8-noeval-nodsmem", "fp64"):
    hp.set_k2_path(path)
    rep = hp.compress(op, t, rank=w.rank, oversample=w.oversample, seed=7)
    ap = sum(p["apply_ms"] for p in rep.report["phases"] if p["phase"] == "h1")
    print(f"{path:12s} K2 {ap:8.1f} ms", flush=True)
hp.set_k2_path("int8")
