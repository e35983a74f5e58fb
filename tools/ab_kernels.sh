#!/bin/bash
# A/B of the D=128 kernel choices through TLATTN_KERNEL (pp = default, 2sm = round-1 pair
# kernel): timings of tools/run_config.py, two rounds. Usage: tools/ab_kernels.sh "pp 2sm" "C5 T0"
KS=${1:-pp 2sm}; CFGS=${2:-C5 T0 C2 C3}
for rep in 1 2; do for kk in $KS; do for c in $CFGS; do
  echo -n "$kk "; TLATTN_KERNEL=$kk timeout 120 python tools/run_config.py $c --iters 12 --time
done; done; done
