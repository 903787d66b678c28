# Builds the sm_100a engine library in-tree (the .so travels to the GPU box with the gpurun
# snapshot). One object per translation unit (make -j builds them in parallel; -MMD tracks
# header dependencies). The oracle (oracle/) is Python/numpy: nothing to compile.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2605_23945_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libtpshift_b200.so
OBJDIR := build/obj
SRCS := abi gemm_tcgen05 gemv decode_ops attention attention_balanced attention_prefill copy persist
OBJS := $(SRCS:%=$(OBJDIR)/%.o)
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

.PHONY: all clean
all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu Makefile
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -MMD -MP -c -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS)
	cat $(OBJDIR)/*.ptxas.log > build_ptxas.log

-include $(OBJS:.o=.d)

clean:
	rm -rf $(LIB) build_ptxas.log $(OBJDIR)



