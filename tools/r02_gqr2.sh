#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02p}
mkdir -p $O
timeout 600 python tools/qr_bench.py 80 64 192:4000 150:6000:4 100:10000:2.5 48:20000 3000:300:5 > $O/qr_bench80.txt 2>&1
timeout 600 python tools/qr_bench.py 42 32 256:3000 128:8000:3 128:8000:2 64:16000:1 30:16000 5000:200:3 > $O/qr_bench42.txt 2>&1
timeout 600 python tools/qr_bench.py 64 48 256:4000 128:8000:4 64:16000 > $O/qr_bench64.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l80.csv python tools/qr_bench.py 80 64 100:10000:2.5 > $O/l80.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l42.csv python tools/qr_bench.py 42 32 128:8000:3 > $O/l42.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l80s.csv python tools/qr_bench.py 80 64 48:20000 > $O/l80s.txt 2>&1
