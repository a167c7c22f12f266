# Build everything in-tree (the .so files travel to the GPU box with gpurun).
#   libsynth.so  : seeded input generator (shared by both sides, no method arithmetic)
#   liboracle.so : the CPU oracle (test infrastructure; plain C, -ffp-contract=off)
#   libtsp.so    : the product: sm_100a CUDA kernels + C-ABI (include/tsp.h)
HOSTCC  := gcc
NVCC    ?= /usr/local/cuda/bin/nvcc
CFLAGS   = -O2 -std=gnu11 -fPIC -Wall -Wno-unused-function
ORCFLAGS = -O2 -std=gnu11 -fPIC -Wall -ffp-contract=off -fno-fast-math
ARCH     = -gencode arch=compute_100a,code=sm_100a
NVFLAGS  = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr

TSP_SRC  = $(wildcard paper_1812_05540_b200/csrc/*.cu)
TSP_HDR  = $(wildcard paper_1812_05540_b200/csrc/*.cuh) include/tsp.h

all: synth oracle oracle_omp tsp
synth: synth/libsynth.so
oracle: oracle/liboracle.so
oracle_omp: oracle/liboracle_omp.so
tsp: paper_1812_05540_b200/libtsp.so

synth/libsynth.so: synth/synth.c
	$(HOSTCC) $(CFLAGS) -fopenmp -shared -o $@ $< -lm

oracle/liboracle.so: $(wildcard oracle/*.c) $(wildcard oracle/*.h)
	$(HOSTCC) $(ORCFLAGS) -shared -o $@ $(wildcard oracle/*.c) -lm

# the same source with its OMP_ROWS loops on all host cores (timing-only oracle row, identical results)
oracle/liboracle_omp.so: $(wildcard oracle/*.c) $(wildcard oracle/*.h)
	$(HOSTCC) $(ORCFLAGS) -fopenmp -shared -o $@ $(wildcard oracle/*.c) -lm

TSP_OBJ  = $(patsubst paper_1812_05540_b200/csrc/%.cu,build/tsp/%.o,$(TSP_SRC))

# one object per translation unit (make -j compiles them in parallel), then one shared library
build/tsp/%.o: paper_1812_05540_b200/csrc/%.cu $(TSP_HDR)
	@mkdir -p build/tsp
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $<

paper_1812_05540_b200/libtsp.so: $(TSP_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(TSP_OBJ) -lcudart

clean:
	rm -rf synth/libsynth.so oracle/liboracle.so oracle/liboracle_omp.so paper_1812_05540_b200/libtsp.so build/tsp

.PHONY: all synth oracle oracle_omp tsp clean
