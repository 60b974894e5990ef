#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02w}
mkdir -p $O
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python tools/qr_bench.py 64 48 256:4000 128:8000:4 64:16000 > $O/qr_bench64.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c5s.csv python tools/one_compress.py c5 131072 > $O/c5s.txt 2>&1
