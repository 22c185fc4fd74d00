# Build of the product library (host C++ + sm_100a CUDA, one .so) and of the
# test-only oracle.  `python -c "import __graft_entry__; __graft_entry__.build()"`
# runs `make -j`.  Host compiler is /usr/bin/g++ (the /opt/gcc wrapper lacks
# libgomp.spec).
CXX      := /usr/bin/g++
NVCC     := /usr/local/cuda/bin/nvcc
PKG      := paper_2303_08394_b200
BUILD    := build
LIBDIR   := $(PKG)/lib
LIB      := $(LIBDIR)/libkifmm_b200.so
ORACLE   := oracle/_build/liboracle.so

CXXFLAGS := -std=c++20 -O3 -march=x86-64-v3 -fPIC -fopenmp -Wall -Wextra -Wno-unused-parameter \
            -Iinclude -I$(PKG)/csrc/host
NVFLAGS  := -std=c++20 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fopenmp -ccbin $(CXX) \
            -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
            -Iinclude -I$(PKG)/csrc/host -I$(PKG)/csrc/cuda -Xptxas -warn-spills

HOST_SRCS := $(wildcard $(PKG)/csrc/host/*.cpp)
CUDA_SRCS := $(wildcard $(PKG)/csrc/cuda/*.cu)
HOST_OBJS := $(patsubst $(PKG)/csrc/host/%.cpp,$(BUILD)/host/%.o,$(HOST_SRCS))
CUDA_OBJS := $(patsubst $(PKG)/csrc/cuda/%.cu,$(BUILD)/cuda/%.o,$(CUDA_SRCS))
HOST_HDRS := $(wildcard $(PKG)/csrc/host/*.hpp) include/kifmm.h
CUDA_HDRS := $(wildcard $(PKG)/csrc/cuda/*.cuh)

.PHONY: all lib oracle clean
all: lib oracle
lib: $(LIB)
oracle: $(ORACLE)

$(BUILD)/host/%.o: $(PKG)/csrc/host/%.cpp $(HOST_HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(HOST_HDRS) $(CUDA_HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(HOST_OBJS) $(CUDA_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) -shared -ccbin $(CXX) -gencode arch=compute_100a,code=sm_100a -o $@ $^ \
	    -cudart static -Xcompiler -fopenmp -ldl -lpthread -lrt

# Test-only oracle: fp64 CPU restatement of SPEC.md (see oracle/oracle.cpp header).
$(ORACLE): oracle/oracle.cpp oracle/oracle.h include/kifmm.h
	@mkdir -p oracle/_build
	$(CXX) -std=c++20 -O3 -march=x86-64-v3 -fPIC -fopenmp -shared -Iinclude -Ioracle $< -o $@

clean:
	rm -rf $(BUILD) $(LIB) oracle/_build
