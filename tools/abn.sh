#!/bin/bash
# Interleaved comparison of several env settings on whole served-mix passes
# (tools/pass_overlap.py: each encoder alone, pairs, all three, whole pass):
#   tools/abn.sh ROUNDS "" "MS_X=1" "MS_Y=2 MS_Z=0" ...
R="$1"; shift
for i in $(seq 1 $R); do
  for SW in "$@"; do
    echo "== [${SW:-default}] round $i"; env $SW python tools/pass_overlap.py 2>&1 | grep -v "^\["
  done
done
