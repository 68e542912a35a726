# Builds the sm_100a product library and the CPU oracle.
NVCC ?= nvcc
PKG := paper_1609_01277_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
LIB := $(PKG)/libosbli.so

all: $(LIB) oracle/liboracle.so

$(CSRC)/kernels.o: $(CSRC)/kernels.cu $(CSRC)/kernels.h $(wildcard $(CSRC)/*.cuh)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; false)

$(CSRC)/api.o: $(CSRC)/api.cpp $(CSRC)/kernels.h include/osbli.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -x cu -c $< -o $@

$(LIB): $(CSRC)/kernels.o $(CSRC)/api.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lnccl -lcudart

oracle/liboracle.so: oracle/oracle.cpp
	g++ -O2 -ffp-contract=off -fno-fast-math -std=c++17 -shared -fPIC $< -o $@

clean:
	rm -f $(CSRC)/*.o $(LIB) oracle/liboracle.so

.PHONY: all clean
