#!/bin/bash
# A/B: L2 bulk-prefetch distance (tiles ahead) for config 4 in place and copy.
mkdir -p gpurun_out
ab() {  # tag env...
  local tag=$1; shift
  env "$@" python bench.py $BARGS --no-e2e --no-cpu > gpurun_out/ab_$tag.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('$tag',d['value'],'ms',d['ms_per_step'],'clk',d['clocks']['sm_mhz'],d['clocks']['reasons'])"
}
for rep in 1 2; do
  for c in c4i c4copy; do
    BARGS="--config $c --steps 10 --warmup 3"
    for pf in 0 592 1184 2368; do ab ${c}_pf${pf}_$rep U16M_PREFETCH=$pf; done
  done
done
