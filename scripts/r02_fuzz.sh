#!/bin/bash
# A long fuzz campaign (20 000 random jobs over every entry point, two seeds).
mkdir -p gpurun_out
for seed in 7 8; do
  U16M_FUZZ_ITERS=10000 U16M_FUZZ_SEED=$seed timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -x > gpurun_out/fuzz_$seed.txt 2>&1
  echo "seed $seed rc=$?" >> gpurun_out/fuzz_summary.txt
done
