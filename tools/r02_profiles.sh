#!/bin/bash
# Round-2 profiles: c3 bench launch list, ncu --set full of K2 (int8, c3 full),
# and of K3 / K4 / K5 on config 5 scaled (the 3D workload where they weigh most)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02g}
mkdir -p $O
N=/usr/local/cuda/bin/ncu
python tools/one_compress.py c5 131072 > $O/c5_plain.txt 2>&1
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c3.log 2>&1
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c5s.csv \
  python tools/one_compress.py c5 131072 > $O/launches_c5s.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on -k regex:sample_apply_i8 --launch-skip 5 -c 1 \
  -o $O/k2i8_c3 python tools/one_compress.py c3 262144 > $O/k2i8.log 2>&1
for k in bsolve_chol_kernel qr_reg_backprop_kernel; do
  timeout 900 $N --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
    -o $O/${k}_c5s python tools/one_compress.py c5 131072 > $O/$k.log 2>&1
done
for f in $O/*.ncu-rep; do $N -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
ls -la $O
