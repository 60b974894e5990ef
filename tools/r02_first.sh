#!/bin/bash
# Round-2 first GPU call: FP64 peaks with a clock record, compute-sanitizer on
# the int8 K2 (small config 3), and the GPU suite as of the round-1 code.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02a
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peaks tools/fp64_peaks.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw --format=csv -lms 200 > $O/fp64_clocks.csv &
SMI=$!
/tmp/fp64_peaks > $O/fp64_peaks.json 2>&1
python tools/dgemm_peak.py >> $O/fp64_peaks.json 2>&1
kill $SMI
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/k2_one_i8.py 4096 > $O/racecheck.txt 2>&1; echo "racecheck rc $?" >> $O/racecheck.txt
timeout 900 compute-sanitizer --tool synccheck python tools/k2_one_i8.py 4096 > $O/synccheck.txt 2>&1; echo "synccheck rc $?" >> $O/synccheck.txt
timeout 900 compute-sanitizer --tool memcheck python tools/k2_one_i8.py 4096 > $O/memcheck.txt 2>&1; echo "memcheck rc $?" >> $O/memcheck.txt
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.txt
