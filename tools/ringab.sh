#!/bin/bash
# Interleaved comparison of env settings on the served path's steady-state
# pass time (tools/ring_rate.py):  tools/ringab.sh ROUNDS "" "MS_X=1" ...
# RR_ARGS="--counts 40 0 0" passes arguments to tools/ring_rate.py
R="$1"; shift
for i in $(seq 1 $R); do
  for SW in "$@"; do
    echo "== [${SW:-default}] round $i $(env $SW python tools/ring_rate.py $RR_ARGS 2>&1 | grep served-path)"
  done
done
