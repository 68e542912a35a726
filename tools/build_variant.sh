#!/bin/bash
# build an experimental variant of libosbli.so: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/.."
NCCL_HOME=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
mkdir -p variants/$1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2 \
  -c paper_1609_01277_b200/csrc/kernels.cu -o variants/$1/kernels.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$1.so variants/$1/kernels.o \
  paper_1609_01277_b200/csrc/api.o paper_1609_01277_b200/csrc/scalar.o paper_1609_01277_b200/csrc/scalar_api.o -L$NCCL_HOME/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL_HOME/lib -lcudart
