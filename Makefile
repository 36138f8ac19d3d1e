# Builds libkvlinc.so (sm_100a) in-tree so it travels with gpurun snapshots.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
PKG := paper_2510_05373_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/libkvlinc.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/kvlc_common.cuh include/kvlinc.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
