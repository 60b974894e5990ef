#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02o}
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l80.csv python tools/qr_bench.py 80 64 100:10000:2.5 > $O/l80.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l42.csv python tools/qr_bench.py 42 32 128:8000:3 > $O/l42.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l80s.csv python tools/qr_bench.py 80 64 48:20000 > $O/l80s.txt 2>&1
