# quick perf check: all configs, kernel only (no e2e / cpu legs)
mkdir -p gpurun_out
for c in ${CONFIGS:-c0 c1 c2 c3 c4i}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err || echo "$c failed"
  python -c "import json;d=json.load(open('gpurun_out/q_$c.json'));r=d['roofline'];print('$c',d['value'],'GB/s in; frac',r['frac'],'kernel_ms',r['kernel_ms'],'clk',d['clocks']['sm_mhz'])"
done
