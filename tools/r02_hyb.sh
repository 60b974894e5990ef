#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r03h}
mkdir -p $O
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
