"""Summarize bench lines (one per config) into the profiles table:
python tools/configs_table.py gpurun_out/r02j/bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    ph = d["report"]["phases"]
    s = lambda k: sum(p.get(k, 0.0) for p in ph)  # noqa: E731
    paths = sorted({p.get("apply_path") for p in ph if p["phase"] == "h1"})
    roof = d["roofline"]
    print(f"{d['config']['description'][:70]:70s} {d['value']:8.4f} s  e2e {d['e2e']['value'] if d.get('e2e') else float('nan'):7.3f}  "
          f"K2 {s('apply_ms'):8.1f} ms ({'/'.join(paths)}, in-step {roof['frac']:.2f}, alone {roof['alone']['frac']:.2f})  "
          f"QR {s('qr_ms'):7.1f}  peel {s('peel_ms'):7.1f}  B {s('bsolve_ms'):7.1f}  "
          f"clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
