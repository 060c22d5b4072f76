# Builds the sm_100a operator library in-tree (it travels to the GPU box
# with the repo snapshot) and the oracle's C restatement.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr
PKG := paper_1903_08243_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/fe_b200.h

all: $(PKG)/libfeb200.so

$(PKG)/libfeb200.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC)

clean:
	rm -f $(PKG)/libfeb200.so

.PHONY: all clean
