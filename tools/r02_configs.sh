#!/bin/bash
# One bench line per BASELINE config (c4 / c5 scaled: their full N needs 8 GPUs)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02j}
mkdir -p $O
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --n 262144 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c4s.json 2> $O/bench_c4s.err
timeout 900 python bench.py --config c5 --n 131072 --steps 3 --warmup 2 --no-cpu --no-e2e > $O/bench_c5s.json 2> $O/bench_c5s.err
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
