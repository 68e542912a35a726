#!/bin/bash
# One GPU round trip used while iterating: parity tests on the production paths
# and the default bench line (plus optional extra bench configs).
#   tools/gpu_check.sh TAG [pytest targets...]   (BENCH_CONFIGS="tgv256_o8 ..." extra lines)
TAG=${1:-x}; shift
TARGETS=${@:-tests/test_gpu_production.py tests/test_gpu_parity.py}
mkdir -p gpurun_out
timeout 900 python -m pytest $TARGETS -x -q -m gpu > gpurun_out/t_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t_$TAG.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err
for c in $BENCH_CONFIGS; do
  timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/b_${TAG}_$c.json 2>> gpurun_out/b_$TAG.err
done
