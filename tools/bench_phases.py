"""Phase sums of bench.py JSON lines: python tools/bench_phases.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    ph = d["report"]["phases"]
    keys = ["apply_ms", "peel_ms", "qr_ms", "bsolve_ms"]
    tot = {k: sum((p.get(k) or 0) for p in ph) for k in keys}
    print(f"{f}: {d['value']:.4f} s  K2 frac {d['roofline']['frac']:.3f}  " + "  ".join(f"{k[:-3]} {v:.1f}" for k, v in tot.items()))
