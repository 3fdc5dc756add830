#!/bin/bash
# Interleaved A/B of an env switch on whole served-mix passes:
#   tools/ab.sh "MS_NO_EARLY_B=1" [rounds]
# runs tools/pass_overlap.py alternately without / with the switch.
SW="$1"; R="${2:-2}"
for i in $(seq 1 $R); do
  echo "== A (default) round $i"; python tools/pass_overlap.py 2>&1 | grep -v "^\[" | tail -4
  echo "== B ($SW) round $i"; env $SW python tools/pass_overlap.py 2>&1 | grep -v "^\[" | tail -4
done
