# Build librotatek.so (sm_100a) and the CPU oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2605_19218_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/rotatek.h

all: $(PKG)/librotatek.so oracle/liboracle.so

# decode_ring.o does not depend on the other decode kernels' headers (and vice versa)
RING_HDR := $(PKG)/csrc/decode_ring.cuh
BASE_HDR := $(filter-out $(RING_HDR),$(HDR))
build/decode_ring.o: $(BASE_HDR) $(RING_HDR)
build/decode.o build/api.o build/calibrate.o build/compress.o build/compress_tc.o build/cov_tc.o build/subspace.o: $(BASE_HDR)

build/%.o: $(PKG)/csrc/%.cu
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/librotatek.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@.tmp $(OBJ) && mv $@.tmp $@

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -fno-fast-math -o $@ $< -lm

clean:
	rm -rf build $(PKG)/librotatek.so oracle/liboracle.so

.PHONY: all clean
