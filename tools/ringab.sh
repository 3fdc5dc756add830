#!/bin/bash
# Interleaved comparison of env settings on the served path's steady-state
# pass time (tools/ring_rate.py):  tools/ringab.sh ROUNDS "" "MS_X=1" ...
R="$1"; shift
for i in $(seq 1 $R); do
  for SW in "$@"; do
    echo "== [${SW:-default}] round $i $(env $SW python tools/ring_rate.py 2>&1 | grep served-path)"
  done
done
