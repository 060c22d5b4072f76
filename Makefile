# Builds the sm_100a operator library in-tree (it travels to the GPU box
# with the repo snapshot) and the oracle's C restatement.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -shared --expt-relaxed-constexpr -lgomp
PKG := paper_1903_08243_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/fe_b200.h

all: $(PKG)/libfeb200.so oracle/liboracle.so oracle/libcpuport.so

# experiment build: make variant V=minb2 FLAGS=-DFE_TENSOR_MINB=2
variant: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) $(FLAGS) -o $(PKG)/libfeb200_$(V).so $(SRC)

oracle: oracle/liboracle.so oracle/libcpuport.so

# the oracle's C restatement (test/baseline infrastructure); the reference's
# BENCH_FLAGS (jit.py:27) with a portable AVX-512 target
oracle/liboracle.so: oracle/fe_oracle.c
	gcc -O3 -march=x86-64-v4 -ffast-math -fopenmp -shared -fPIC -o $@ $< -lm

# the SIMD-batched CPU port (cpu_baseline / reference arm; baseline infrastructure)
oracle/libcpuport.so: oracle/fe_cpu_port.cpp
	g++ -O3 -march=x86-64-v4 -ffast-math -fopenmp -std=c++17 -shared -fPIC -o $@ $<

$(PKG)/libfeb200.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC)

clean:
	rm -f $(PKG)/libfeb200.so oracle/liboracle.so oracle/libcpuport.so

.PHONY: all clean oracle variant
