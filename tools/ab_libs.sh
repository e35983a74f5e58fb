#!/bin/bash
# A/B of library variants built into build/lib<name>.so: parity (tests/test_parity_gpu.py) for each non-base
# variant, then two rounds of tools/run_config.py timings. Usage: tools/ab_libs.sh "base v1 v2" "T0 C5"
# usage: build/ab.sh "libA libB ..." "cfgs" ; parity (tests/test_parity_gpu.py) for each non-base lib, then A/B timing
LIBS=$1; CFGS=${2:-T0 C2 C3 C5}
for lib in $LIBS; do
  if [ "$lib" != "base" ]; then
    echo "== parity $lib"; TLATTN_LIB=build/lib$lib.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
  fi
done
for rep in 1 2; do for lib in $LIBS; do for c in $CFGS; do
  echo -n "$lib "; TLATTN_LIB=build/lib$lib.so timeout 120 python tools/run_config.py $c --iters 12 --time
done; done; done
