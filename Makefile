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

# the SpMV kernel variants are separate units (spmv_inst_*.cu): build them in parallel
MAKEFLAGS += -j$(shell nproc 2>/dev/null || echo 8)

.PHONY: all lib oracle cpp probe clean
all: lib oracle

lib: $(PKG)/libcsr5g.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DCSR5G_BUILD -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(PKG)/libcsr5g.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xcompiler -fPIC -Xlinker -soname=libcsr5g.so $(OBJS) -o $@

oracle:
	$(MAKE) -C oracle

# C++ drop-in (include/csr5/*.hpp) through the CMake package (cmake/); the
# programs need a GPU to run (tests/test_gpu_cpp.py)
cpp: $(PKG)/libcsr5g.so
	cmake -S tests/cpp -B build/cpp -Dcsr5_DIR=$(CURDIR)/cmake && cmake --build build/cpp

# measurement tool (random-gather ceiling), not part of the product
probe: build/gather_probe
build/gather_probe: tools/gather_probe.cu
	@mkdir -p build
	$(NVCC) -O3 -std=c++17 $(ARCH) $< -o $@

clean:
	rm -rf build $(PKG)/libcsr5g.so
	$(MAKE) -C oracle clean
