#!/bin/bash
# GPU-side A/B driver: tools/ab_run.sh OUT "orders" variant names... (cur = default build)
out=$1; orders=$2; shift 2
mkdir -p gpurun_out
for o in $orders; do
  timeout 300 bash tools/ab.sh 256 $o "$@" >> gpurun_out/$out 2>&1
done
