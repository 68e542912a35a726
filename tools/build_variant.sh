#!/bin/bash
# Build an experimental variant of libosbli.so with extra nvcc flags:
#   tools/build_variant.sh NAME "-DFOO=1 ..." [orders-to-build, default "1 2 3 4 5 6"]
# -> variants/lib_NAME.so (select it with OSBLI_LIB=variants/lib_NAME.so)
set -e
cd "$(dirname "$0")/.."
NCCL_HOME=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2"
D=variants/$1
mkdir -p $D
MS=${3:-"1 2 3 4 5 6"}
pids=()
for m in $MS; do
  nvcc $FL -DOSBLI_M=$m -Xptxas -v -c paper_1609_01277_b200/csrc/kernels_order.cu -o $D/kernels_m$m.o 2> $D/ptxas_m$m.log &
  pids+=($!)
done
nvcc $FL -c paper_1609_01277_b200/csrc/kernels.cu -o $D/kernels.o &
pids+=($!)
for p in "${pids[@]}"; do wait $p; done
# orders not rebuilt come from the default build
objs=""
for m in 1 2 3 4 5 6; do
  if [ -f $D/kernels_m$m.o ] && [[ " $MS " == *" $m "* ]]; then objs="$objs $D/kernels_m$m.o"; else objs="$objs paper_1609_01277_b200/csrc/kernels_m$m.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$1.so $D/kernels.o $objs \
  paper_1609_01277_b200/csrc/api.o paper_1609_01277_b200/csrc/scalar.o paper_1609_01277_b200/csrc/scalar_api.o \
  -L$NCCL_HOME/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL_HOME/lib -lcudart
echo built variants/lib_$1.so
