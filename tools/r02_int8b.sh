#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02f}
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_k2_int8.py tests/test_gpu_k2.py -m gpu -q -s -p no:cacheprovider > $O/pytest_int8.txt 2>&1; echo "pytest rc $?" >> $O/pytest_int8.txt
