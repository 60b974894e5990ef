#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02c
mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 3000 python -m pytest tests/test_gpu_shard.py tests/test_gpu_fullsize.py tests/test_gpu_callback.py tests/test_shim.py -m gpu -q -x --timeout 1800 -p no:cacheprovider -s > $O/pytest_new.txt 2>&1; echo "pytest rc $?" >> $O/pytest_new.txt
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > $O/bench_c1_ours.json 2> $O/bench_c1_ours.err
timeout 900 python bench.py --config c1 --impl reference --steps 3 --warmup 1 > $O/bench_c1_ref.json 2> $O/bench_c1_ref.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_c3_ref.json 2> $O/bench_c3_ref.err
