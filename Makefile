# Builds the sm_100a C-ABI library of the hot path (no GPU needed to compile).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DHOLO_WITH_NCCL --expt-relaxed-constexpr $(EXTRA)
SRC := paper_1904_04884_b200/csrc/kernels.cu paper_1904_04884_b200/csrc/prox_strip.cu paper_1904_04884_b200/csrc/engine.cu paper_1904_04884_b200/csrc/segment.cu paper_1904_04884_b200/csrc/synth.cu paper_1904_04884_b200/csrc/peer.cu paper_1904_04884_b200/csrc/gfft.cu
HDR := $(wildcard paper_1904_04884_b200/csrc/*.cuh) include/holo_b200.h
LIB := paper_1904_04884_b200/libholo_b200.so
OBJ := $(patsubst paper_1904_04884_b200/csrc/%.cu,build/%.o,$(SRC))

CLIB := paper_1904_04884_b200/libholo_b200_checked.so
COBJ := $(patsubst paper_1904_04884_b200/csrc/%.cu,build/checked/%.o,$(SRC))

all: $(LIB)

# bounds-checked build (HOLO_CHECKS, common.cuh): tests/test_gpu_checked.py
checked: $(CLIB)

build/checked/%.o: paper_1904_04884_b200/csrc/%.cu $(HDR)
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DHOLO_CHECKS -c $< -o $@

$(CLIB): $(COBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(COBJ) -ldl

build/%.o: paper_1904_04884_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ) -ldl

clean:
	rm -rf build $(LIB) $(CLIB)

.PHONY: all checked clean
