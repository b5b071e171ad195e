# Builds the product library (sm_100a only) and the test oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr
PKG := paper_2503_01471_b200
SRC := $(PKG)/csrc/blas.cu $(PKG)/csrc/tlas.cu $(PKG)/csrc/cast.cu \
       $(PKG)/csrc/checksum.cu $(PKG)/csrc/sim.cu $(PKG)/csrc/abi.cu
HDR := $(PKG)/csrc/agr_internal.cuh include/agr.h include/agr_sim.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/lib/libagr.so

all: $(LIB) oracle/liboracle.so tools/fma_peak

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -lrt -ldl -lpthread

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	gcc -O2 -std=c11 -fPIC -shared -pthread -Wall -o $@ oracle/oracle.c -lm

tools/fma_peak: tools/fma_peak.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $(PKG)/csrc/cast.cu -o /dev/null

clean:
	rm -rf build $(LIB) oracle/liboracle.so tools/fma_peak

.PHONY: all clean ptxas
