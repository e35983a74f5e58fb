#!/bin/bash
# Repeated launches of one library variant on one config (hang / trap check + timing).
# usage: build/stress.sh lib cfg n
for i in $(seq 1 $3); do TLATTN_LIB=build/lib$1.so timeout 120 python tools/run_config.py $2 --iters 30 --time 2>&1 | grep -E "TFLOP|Error" | head -1; done
