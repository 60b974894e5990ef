#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02r}
mkdir -p $O
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
