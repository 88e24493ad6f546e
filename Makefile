# Top-level build.  Everything lands in-tree so gpurun ships it to the GPU box.
#   paper_1503_05032_b200/libcsr5g.so   the product (sm_100a, static cudart)
#   oracle/liboracle.so, oracle/_ref/   test infrastructure (oracle/Makefile)
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
            -Xptxas -v -cudart static --expt-relaxed-constexpr
PKG      := paper_1503_05032_b200
SRCS     := $(wildcard $(PKG)/csrc/*.cu)
OBJS     := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/csr5g.h

.PHONY: all lib oracle shim probe clean
all: lib oracle

lib: $(PKG)/libcsr5g.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DCSR5G_BUILD -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(PKG)/libcsr5g.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC $(OBJS) -o $@

oracle:
	$(MAKE) -C oracle

# C++ drop-in shim test (include/csr5g.hpp); needs a GPU to run
CXX_SYS  := $(if $(wildcard /usr/bin/g++),/usr/bin/g++,g++)
shim: build/shim_test
build/shim_test: tests/cpp/shim_test.cpp include/csr5g.hpp include/csr5g.h $(PKG)/libcsr5g.so
	@mkdir -p build
	$(CXX_SYS) -std=c++20 -O2 -Wall -pthread -Iinclude $< -L$(PKG) -lcsr5g \
	  -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

# measurement tool (random-gather ceiling), not part of the product
probe: build/gather_probe
build/gather_probe: tools/gather_probe.cu
	@mkdir -p build
	$(NVCC) -O3 -std=c++17 $(ARCH) $< -o $@

clean:
	rm -rf build $(PKG)/libcsr5g.so
	$(MAKE) -C oracle clean
