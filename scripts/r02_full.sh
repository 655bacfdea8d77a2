#!/bin/bash
# Round-2 full GPU pass: smoke, the whole -m gpu suite, the default bench line
# twice (e2e spread), the reference arm, and the per-config quick numbers.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
for i in 1 2; do python bench.py > gpurun_out/bench_default_$i.json 2> gpurun_out/bench_default_$i.err; done
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CONFIGS="c0 c1 c2 c3" bash scripts/quick.sh > gpurun_out/quick.txt 2>&1
