#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02s}
mkdir -p $O
timeout 600 python tools/qr_bench.py 80 64 192:4000 150:6000:4 100:10000:2.5 48:20000 3000:300:5 > $O/qr_bench80.txt 2>&1
timeout 600 python tools/qr_bench.py 42 32 256:3000 128:8000:3 128:8000:2 64:16000:1 30:16000 5000:200:3 > $O/qr_bench42.txt 2>&1
timeout 600 python tools/qr_bench.py 64 48 256:4000 128:8000:4 64:16000 > $O/qr_bench64.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l42.csv python tools/qr_bench.py 42 32 128:8000:3 > $O/l42.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l80s.csv python tools/qr_bench.py 80 64 48:20000 > $O/l80s.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "3d_multilevel" > $O/pytest_3d.txt 2>&1; echo "rc $?" >> $O/pytest_3d.txt
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
