#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02i}
mkdir -p $O
timeout 4000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1800 > $O/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.txt
N=/usr/local/cuda/bin/ncu
for k in bsolve_chol_kernel qr_reg_backprop_kernel; do
  timeout 900 $N --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
    -o $O/${k}_c5s python tools/one_compress.py c5 131072 > $O/$k.log 2>&1
done
for f in $O/*.ncu-rep; do $N -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
