#!/bin/bash
# Per-kernel durations of one bench config under ncu (launch list only, caches NOT flushed between
# kernels so metadata produced by a pre-pass stays warm as in the real step).
# usage: CFG=c3 TAG=x bash scripts/ncu_launches.sh ; prints kernel name + median duration
C=${CFG:-c1}; T=${TAG:-$C}
CMD="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/nl_$T.csv $CMD > /dev/null 2>&1
python - gpurun_out/nl_$T.csv $T <<'PY'
import csv, sys, statistics, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ik].split('(')[0][:60]].append(float(r[iv].replace(',', '')))
for k, v in d.items():
    print(sys.argv[2], f"{k:60s} n={len(v):3d} median={statistics.median(v)/1e3:8.1f} us")
PY
