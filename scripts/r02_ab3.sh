#!/bin/bash
# A/B: batched (config 3) with the table fill as a PDL primary kernel (new)
# vs cudaMemsetAsync (ab/libu16m_old.so), same box, alternating; then the
# batched parity tests on the new build.
mkdir -p gpurun_out
for rep in 1 2 3; do
  echo "== old $rep"; U16M_LIBRARY=$PWD/ab/libu16m_old.so python scripts/batched_probe.py
  echo "== new $rep"; python scripts/batched_probe.py
done
python -m pytest tests -m gpu -q -x -k "batched or c3 or config3" 2>&1 | tail -3
