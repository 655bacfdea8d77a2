#!/bin/bash
# ncu --set full with source counters (per-SASS executed instructions) of the
# config-4 in-place and copy repair kernels.
mkdir -p gpurun_out
for c in c4i c4copy; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu --set full --section SourceCounters --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_src_$c $CMD > gpurun_out/ncu_src_$c.log 2>&1
  echo "ncu $c rc=$?" >> gpurun_out/ncu_src_rc.txt
done
