#!/bin/bash
# Host pipeline chunk-size / ramp sweep (config 1), two interleaved passes.
export MODES=${MODES:-inplace,copy}
for rep in 1 2; do
  for r in 0 1; do
    for c in ${CHUNKS:-16384 32768 65536}; do
      U16M_PIPE_RAMP=$r U16M_PIPE_CHUNK_KIB=$c python scripts/e2e_probe.py | sed "s/^/rep$rep ramp$r chunk$c /"
    done
  done
done
