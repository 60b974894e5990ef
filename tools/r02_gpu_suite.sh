#!/bin/bash
# GPU suite + smoke + a short c3 bench (round 2 iteration)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r02b}
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc $?" >> $O/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} > $O/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc $?" >> $O/bench.err
