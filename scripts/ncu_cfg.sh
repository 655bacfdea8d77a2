# ncu launch list + one full capture of the top repair kernel for config $CFG (1 GPU).
# usage: CFG=c2 KREGEX=repair bash scripts/ncu_cfg.sh
mkdir -p gpurun_out
C=${CFG:-c1}; K=${KREGEX:-repair}; T=${TAG:-$C}
CMD="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_$T.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_launch_$T.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$T $CMD > gpurun_out/ncu_full_$T.log 2>&1
echo "ncu $T rc=$?"
