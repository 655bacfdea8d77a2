#!/bin/bash
# Round-end evidence (1 GPU): default bench line, reference arm, all configs, and the ncu launch
# list of the default bench command (fewer steps). Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
bash scripts/quick.sh > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv \
  python bench.py --steps 5 --warmup 3 > gpurun_out/ncu_default.log 2>&1; echo "ncu rc=$?"
