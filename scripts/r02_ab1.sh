#!/bin/bash
# A/B: small-job tile size for config 0, in-place write-back granularity for
# config 4, then the whole GPU test suite.
mkdir -p gpurun_out
ab() {  # name env... -- bench args
  local tag=$1; shift
  env "$@" python bench.py $BARGS --no-e2e --no-cpu > gpurun_out/ab_$tag.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));print('$tag',d['value'],'ms',d['ms_per_step'],'clk',d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  BARGS="--config c0 --steps 50 --warmup 5"
  ab c0_sv0_$rep U16M_SMALL_SV=0
  ab c0_sv4_$rep U16M_SMALL_SV=4
  ab c0_sv46_$rep U16M_SMALL_SV=46
  ab c0_sv28_$rep U16M_SMALL_SV=28
done
for rep in 1 2; do
  BARGS="--config c4i --steps 10 --warmup 3"
  for g in 1 2 4 8; do ab c4i_g${g}_$rep U16M_GRAN=$g; done
done
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
