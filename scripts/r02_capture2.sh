#!/bin/bash
# Round-2 capture with the final code: default bench line, reference arm,
# launch list of the default command, ncu --set full of the batched (C3)
# repair kernel and of the read-only validation kernel on C4.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default_final.csv python bench.py > gpurun_out/ncu_default_final.log 2>&1
echo "ncu default rc=$?" >> gpurun_out/ncu_rc2.txt
CMD="python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batched_tile_kernel -s 3 -c 1 -o gpurun_out/prof_c3_r02 $CMD > gpurun_out/ncu_full_c3_r02.log 2>&1
echo "ncu c3 rc=$?" >> gpurun_out/ncu_rc2.txt
timeout 900 ncu --set full --clock-control none -k regex:stream_kernel -c 1 -o gpurun_out/prof_count_c4 python scripts/count_probe.py > gpurun_out/ncu_count.log 2>&1
echo "ncu count rc=$?" >> gpurun_out/ncu_rc2.txt
