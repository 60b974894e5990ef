#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02e}
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc $?" >> $O/smoke.txt
timeout 1800 python -m pytest tests/test_gpu_fullsize.py::test_full_c3_int8_samples_match_fp64_and_host tests/test_gpu_k2_int8.py -m gpu -q -x -s -p no:cacheprovider > $O/pytest_int8.txt 2>&1; echo "pytest rc $?" >> $O/pytest_int8.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc $?" >> $O/bench.err
