# Build of the sm_100a CUDA library (C ABI in include/lcnn_cuda.h).
# `make -j` here cross-compiles without a GPU; __graft_entry__.build() runs it.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -warn-spills --expt-relaxed-constexpr
PKG     := paper_1610_03618_b200
SRC     := $(PKG)/csrc
OBJDIR  := build/obj
CU      := transform pool softmax gemm conv capi
OBJS    := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU)))
LIB     := $(PKG)/lib/liblcnn_cuda.so

all: $(LIB) oracle

$(OBJDIR)/%.o: $(SRC)/%.cu $(SRC)/common.cuh $(SRC)/internal.h $(SRC)/tc.cuh $(SRC)/tc_gemm.cuh include/lcnn_cuda.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
