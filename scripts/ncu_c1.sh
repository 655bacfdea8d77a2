# launch list + full capture of the repair kernel on config 1 (1 GPU).
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-c1} --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_${CFG:-c1}.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG:-c1}.csv $CMD > gpurun_out/ncu_launch_${CFG:-c1}.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:repair_kernel -s 3 -c 1 -o gpurun_out/prof_${CFG:-c1} $CMD > gpurun_out/ncu_full_${CFG:-c1}.log 2>&1
echo "ncu rc=$?"
