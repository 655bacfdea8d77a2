#!/bin/bash
# Round-2 final capture (final code): the driver's order (reference arm first,
# then the default bench line), two more default lines for the spread, the
# per-config quick numbers, the launch list of the default command and one
# ncu --set full capture per headline / parity kernel.
mkdir -p gpurun_out/final
O=gpurun_out/final
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for i in 1 2 3; do python bench.py > $O/bench_default_$i.json 2> $O/bench_default_$i.err; done
CONFIGS="c0 c1 c2 c3" bash scripts/quick.sh > $O/quick.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default_cmd.csv python bench.py > $O/ncu_default.log 2>&1
echo "ncu default rc=$?" >> $O/ncu_rc.txt
for c in c4copy c4i c3; do
  K=stream_kernel; [ $c = c3 ] && K=batched_tile_kernel
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $O/prof_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_$c.log 2>&1
  echo "ncu $c rc=$?" >> $O/ncu_rc.txt
done
timeout 900 ncu --set full --clock-control none -k regex:stream_kernel -s 1 -c 1 -o $O/prof_count_c4 python scripts/count_probe.py > $O/ncu_count.log 2>&1
echo "ncu count rc=$?" >> $O/ncu_rc.txt
# keep gpurun_out small (the merge-back limit is 64 MiB): text summaries only
for r in $O/prof_*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; done
python scripts/launch_summary.py $O/launches_default_cmd.csv > $O/launches_default_cmd_summary.txt 2>&1
rm -f $O/prof_*.ncu-rep
