# Builds everything in-tree (the .so files travel to the GPU box with gpurun):
#   paper_2411_19419_b200/libspconv_b200.so  -- the product: sm_100a kernels + C ABI
#   oracle/_build, oracle/_ref               -- the parity checkers (oracle/Makefile)
#   tests/cpp/_build/test_dropin             -- drop-in C++ API test program
#   tools/_build/spconv_b200                 -- the command-line front end (build/convolve/verify/nnz/bench)
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     ?= g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-Wall -Xptxas -v --expt-relaxed-constexpr
PKG     := paper_2411_19419_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRCS))
LIB     := $(PKG)/libspconv_b200.so

all: $(LIB) oracle dropin cli

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

build/obj/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/internal.h $(wildcard $(PKG)/csrc/*.cuh) include/spconv_b200.h
	@mkdir -p build/obj build/ptxas
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/ptxas/$*.log || (cat build/ptxas/$*.log; false)

oracle:
	$(MAKE) --no-print-directory -C oracle

dropin: tests/cpp/_build/test_dropin

tests/cpp/_build/test_dropin: tests/cpp/test_dropin.cpp $(wildcard include/spconv/*.hpp) include/spconv_b200.h $(LIB)
	@mkdir -p tests/cpp/_build
	$(CXX) -O2 -std=c++20 -Wall -Wextra -Iinclude -o $@ $< -L$(PKG) -lspconv_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

cli: tools/_build/spconv_b200

tools/_build/spconv_b200: tools/spconv_b200_cli.cpp $(wildcard include/spconv/*.hpp) include/spconv_b200.h $(LIB)
	@mkdir -p tools/_build
	$(CXX) -O2 -std=c++20 -Wall -Wextra -Iinclude -o $@ $< -L$(PKG) -lspconv_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

clean:
	rm -rf build $(LIB) tests/cpp/_build tools/_build
	$(MAKE) -C oracle clean

.PHONY: all oracle dropin cli clean
