"""Print value, setup time and per-phase (level, host wait, device ms) of bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            r = d["report"]
            print(f, d["value"], "setup_ms", r.get("setup_ms"),
                  [(p["phase"][0] + str(p["level"]), p.get("host_wait_ms"), p["wall_ms_total"]) for p in r["phases"]])
