#!/bin/bash
# A/B timing of two library builds on the same box: tools/ab_configs.sh LIB_A LIB_B [configs...]
A=$1; B=$2; shift 2
CFGS=${@:-T0 C2 C3 C5}
for rep in 1 2; do
  for lib in $A $B; do
    for c in $CFGS; do
      echo -n "$(basename $lib) "; TLATTN_LIB=$lib python tools/run_config.py $c --iters 12 --time
    done
  done
done
