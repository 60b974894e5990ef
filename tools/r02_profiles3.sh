#!/bin/bash
# Round-2 final launch lists (same commands as the bench lines) and ncu --set
# full captures of the K4 Gram / apply kernels and the K5 Gram kernel.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r03q}
mkdir -p $O
N=/usr/local/cuda/bin/ncu
python tools/one_compress.py c4 262144 > $O/c4s_plain.txt 2>&1
timeout 1200 $N --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c3.log 2>&1
timeout 1200 $N --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c5s.csv \
  python tools/one_compress.py c5 131072 > $O/launches_c5s.log 2>&1
timeout 1200 $N --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c4s.csv \
  python tools/one_compress.py c4 262144 > $O/launches_c4s.log 2>&1
cap() {  # name regex skip config n
  timeout 900 $N --set full --clock-control none --import-source on -k regex:$2 --launch-skip $3 -c 1 \
    -o $O/$1 python tools/one_compress.py $4 $5 > $O/$1.log 2>&1
}
cap k2fp64_c4s 'sample_apply_kernel' 2 c4 262144
cap gqr_gram_c5s 'gqr_gram_kernel' 15 c5 131072
cap gqr_apply_c5s 'gqr_apply_kernel' 15 c5 131072
cap k5_gram_c5s '^gram_kernel|::gram_kernel' 4 c5 131072
for f in $O/*.ncu-rep; do $N -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
rm -f $O/*.ncu-rep
ls -la $O
