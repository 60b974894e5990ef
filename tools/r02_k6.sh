#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02z}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
HP_PLAN_TIMING=1 timeout 900 python bench.py --config c5 --n 131072 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
nproc > $O/nproc.txt
