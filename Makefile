# Build of the sm_100a CUDA library (C ABI in include/lcnn_cuda.h).
# `make -j` here cross-compiles without a GPU; __graft_entry__.build() runs it.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) $(if $(filter 1,$(PROFILING)),-DLCNN_PROFILING_KNOBS) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -warn-spills --expt-relaxed-constexpr $(EXTRA_NVFLAGS)
PKG     := paper_1610_03618_b200
SRC     := $(PKG)/csrc
OBJDIR  := build/obj
CU      := transform pool softmax gemm conv capi
OBJS    := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU)))
LIB     := $(PKG)/lib/liblcnn_cuda.so
# C++ drop-in host API (lcnn:: of the reference headers) over the C ABI
CXX     ?= g++
CUDA    ?= /usr/local/cuda
HOSTSRC := $(wildcard $(PKG)/host/src/*.cpp)
HOSTOBJ := $(patsubst $(PKG)/host/src/%.cpp,$(OBJDIR)/host_%.o,$(HOSTSRC))
HOSTLIB := $(PKG)/lib/liblcnn.so
HOSTFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -I$(PKG)/host/include -Iinclude -I$(CUDA)/include

TOOLS   := build/tools/calibrate_b200 build/tools/lcnn

all: $(LIB) $(HOSTLIB) $(TOOLS) oracle

build/tools/%: tools/%.cpp $(HOSTLIB)
	@mkdir -p build/tools
	$(CXX) $(HOSTFLAGS) $< -o $@ -L$(PKG)/lib -llcnn -llcnn_cuda \
	  -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib'

$(OBJDIR)/host_%.o: $(PKG)/host/src/%.cpp $(wildcard $(PKG)/host/include/lcnn/*.hpp) $(PKG)/host/src/json_lite.hpp include/lcnn_cuda.h include/lcnn_net.h
	@mkdir -p $(OBJDIR)
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(HOSTLIB): $(HOSTOBJ) $(LIB)
	$(CXX) -shared -o $@ $(HOSTOBJ) -L$(PKG)/lib -llcnn_cuda -Wl,-rpath,'$$ORIGIN' \
	  -L$(CUDA)/lib64 -lcudart_static -lpthread -ldl -lrt

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
