#!/bin/bash
# Round-2 GPU capture: parity suite, batched decomposition, per-config quick
# numbers, ncu full captures of the config-4 copy / in-place kernels and the
# launch list of the default bench command.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
python scripts/batched_probe.py > gpurun_out/batched_probe.txt 2>&1
CONFIGS="c0 c1 c2 c3" bash scripts/quick.sh > gpurun_out/quick.txt 2>&1
for c in c4copy c4i; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_$c $CMD > gpurun_out/ncu_full_$c.log 2>&1
  echo "ncu $c rc=$?" >> gpurun_out/ncu_rc.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default_cmd.csv python bench.py > gpurun_out/ncu_default.log 2>&1
echo "ncu default rc=$?" >> gpurun_out/ncu_rc.txt
