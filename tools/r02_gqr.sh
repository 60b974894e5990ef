#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02n}
mkdir -p $O
for mode in gram householder; do
  export HP_QR=$mode
  timeout 600 python tools/qr_bench.py 80 64 192:4000 150:6000:4 100:10000:2.5 48:20000 3000:300:5 > $O/qr_bench80_$mode.txt 2>&1
  timeout 600 python tools/qr_bench.py 42 32 256:3000 128:8000:3 128:8000:2 64:16000:1 30:16000 5000:200:3 > $O/qr_bench42_$mode.txt 2>&1
  timeout 600 python tools/qr_bench.py 64 48 256:4000 128:8000:4 64:16000 > $O/qr_bench64_$mode.txt 2>&1
done
unset HP_QR
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_shard.py -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
