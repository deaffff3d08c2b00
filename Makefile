# Builds the sm_100a CUDA library (libgvp_b200.so) in-tree and the oracle's
# reference build (oracle/_ref, only where /root/reference exists).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2411_03416_b200/csrc/*.cu)
HDR := $(wildcard paper_2411_03416_b200/csrc/*.cuh) include/gvp_b200.h
LIB := paper_2411_03416_b200/libgvp_b200.so
OBJ := $(patsubst paper_2411_03416_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB)

build/%.o: paper_2411_03416_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -Xcompiler -fPIC

oracle:
	oracle/build_ref.sh

clean:
	rm -rf build $(LIB)

.PHONY: all clean oracle
