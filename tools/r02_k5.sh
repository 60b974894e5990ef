#!/bin/bash
# c4 / c5 scaled bench lines + the parity tests that exercise K2 / K4 / K5
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02x}
mkdir -p $O
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
