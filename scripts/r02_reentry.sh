#!/bin/bash
# Re-entry check of the restored tree: smoke, full GPU suite, default bench line.
mkdir -p gpurun_out/reentry
O=gpurun_out/reentry
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
cat $O/bench_default.json
CONFIGS="c0 c1 c2 c3" bash scripts/quick.sh > $O/quick.txt 2>&1
cat $O/quick.txt | tail -20
