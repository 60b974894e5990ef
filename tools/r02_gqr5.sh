#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02t}
mkdir -p $O
for th in 1e-7 1e-9; do
HP_GQR_THETA=$th HP_GQR_STAGES=7 timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "3d_multilevel and c5" > $O/pytest_3d_$th.txt 2>&1; echo "rc $?" >> $O/pytest_3d_$th.txt
done
HP_QR=householder timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s -p no:cacheprovider -k "3d_multilevel and c5" > $O/pytest_3d_hh.txt 2>&1
