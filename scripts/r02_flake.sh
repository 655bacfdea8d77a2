#!/bin/bash
# Repeat the batched host helper to look for intermittent mismatches.
mkdir -p gpurun_out
fails=0
for i in $(seq 1 25); do
  python tests/gpu_helpers/batched_host_check.py > /tmp/bh_$i.txt 2>&1 || { fails=$((fails+1)); tail -2 /tmp/bh_$i.txt >> gpurun_out/flake.txt; }
done
echo "batched host helper: $fails failures in 25 runs" >> gpurun_out/flake.txt
