#!/bin/bash
# A/B of kernel knobs on one config: VARIANTS is a list of "NAME=VALUE[,NAME=VALUE]" (or "base").
# Usage: CFG=c1 VARIANTS="base U16M_PREFETCH=0" bash scripts/ab_env.sh
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do
  for v in ${VARIANTS:-base}; do
    envs=""; [ "$v" != base ] && envs=$(echo "$v" | tr ',' ' ')
    out=$(env $envs timeout 300 python bench.py --config ${CFG:-c1} --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e 2>/dev/null |
      python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['roofline']['kernel_ms'],d['clocks']['sm_mhz'])")
    echo "rep$rep ${CFG:-c1} $v $out"
  done
done
