# Builds the sm_100a product library and the CPU oracle.
NVCC ?= nvcc
PKG := paper_1609_01277_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
LIB := $(PKG)/libosbli.so
# NCCL: the copy torch loads (pip nvidia-nccl), so that one libnccl.so.2 serves
# both torch and libosbli in a process regardless of import order
NCCL_HOME ?= $(shell python -c "import nvidia.nccl as n; print(list(n.__path__)[0])" 2>/dev/null)
ifneq ($(NCCL_HOME),)
NCCL_INC := -I$(NCCL_HOME)/include
NCCL_LIB := -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_HOME)/lib
else
NCCL_INC :=
NCCL_LIB := -lnccl
endif

all: $(LIB) oracle/liboracle.so

KHDR := $(CSRC)/kernels.h $(CSRC)/dispatch.h $(wildcard $(CSRC)/*.cuh)
# order-dependent kernels: one object per stencil half width M (built in parallel)
KM_OBJS := $(foreach m,1 2 3 4 5 6,$(CSRC)/kernels_m$(m).o)

$(CSRC)/kernels_m%.o: $(CSRC)/kernels_order.cu $(KHDR)
	$(NVCC) $(NVFLAGS) -DOSBLI_M=$* -c $< -o $@ 2> $(CSRC)/ptxas_m$*.log || (cat $(CSRC)/ptxas_m$*.log; false)

$(CSRC)/kernels.o: $(CSRC)/kernels.cu $(KHDR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; false)

$(CSRC)/api.o: $(CSRC)/api.cpp $(CSRC)/kernels.h $(CSRC)/dispatch.h $(CSRC)/weights.h include/osbli.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC $(NCCL_INC) -x cu -c $< -o $@

$(CSRC)/scalar.o: $(CSRC)/scalar.cu $(CSRC)/scalar.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas_scalar.log || (cat $(CSRC)/ptxas_scalar.log; false)

$(CSRC)/scalar_api.o: $(CSRC)/scalar_api.cpp $(CSRC)/scalar.h $(CSRC)/weights.h include/osbli.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -x cu -c $< -o $@

$(LIB): $(CSRC)/kernels.o $(KM_OBJS) $(CSRC)/api.o $(CSRC)/scalar.o $(CSRC)/scalar_api.o
	$(NVCC) $(ARCH) -shared -o $@ $^ $(NCCL_LIB) -lcudart

oracle/liboracle.so: oracle/oracle.cpp
	g++ -O2 -ffp-contract=off -fno-fast-math -std=c++17 -shared -fPIC $< -o $@

clean:
	rm -f $(CSRC)/*.o $(LIB) oracle/liboracle.so

.PHONY: all clean
