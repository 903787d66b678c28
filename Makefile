# Builds the sm_100a engine library in-tree (the .so travels to the GPU box with
# the gpurun snapshot). The oracle (oracle/) is Python/numpy: nothing to compile.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2605_23945_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libtpshift_b200.so
SRCS := $(CSRC)/abi.cu $(CSRC)/gemm_tcgen05.cu $(CSRC)/decode_ops.cu $(CSRC)/attention.cu $(CSRC)/attention_balanced.cu $(CSRC)/attention_prefill.cu $(CSRC)/copy.cu
HDRS := $(CSRC)/common.cuh $(CSRC)/decode_ops.cuh $(CSRC)/attention_common.cuh include/tpshift_b200.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

.PHONY: all clean
all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f $(LIB) build_ptxas.log
