#!/bin/bash
# Round-2 final evidence: smoke, the GPU suite, one bench line per config (both
# arms for c1 and c3), K4 micro-benchmark on both implementations.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${1:-r03z}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
bash tools/r02_configs.sh ${1:-r03z}
timeout 900 python bench.py --impl reference --config c1 --steps 3 --warmup 1 > $O/bench_ref_c1.json 2> $O/bench_ref_c1.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err
if [ -n "$QR_BENCH" ]; then
for mode in gram householder; do
  export HP_QR=$mode
  timeout 600 python tools/qr_bench.py 80 64 192:4000 150:6000:4 100:10000:2.5 48:20000 3000:300:5 > $O/qr_bench80_$mode.txt 2>&1
  timeout 600 python tools/qr_bench.py 42 32 256:3000 128:8000:3 128:8000:2 64:16000:1 30:16000 5000:200:3 > $O/qr_bench42_$mode.txt 2>&1
  timeout 600 python tools/qr_bench.py 64 48 256:4000 128:8000:4 64:16000 4000:400:4 > $O/qr_bench64_$mode.txt 2>&1
done
unset HP_QR
fi
