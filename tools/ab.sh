#!/bin/bash
# A/B device timing of variant libraries: tools/ab.sh N ORDER name1 name2 ... (cur = default build)
# REPS (default 3) interleaved repetitions of STEPS (default 40) RK3 steps each
n=$1; o=$2; shift 2
for rep in $(seq 1 ${REPS:-3}); do
  for v in "$@"; do
    if [ "$v" = cur ]; then lib=""; else lib=variants/lib_$v.so; fi
    OSBLI_LIB=$lib python tools/quickbench.py $n $o ${STEPS:-40} 2>&1 | tail -1
  done
done
