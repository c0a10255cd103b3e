# Builds every native artefact in-tree (the .so files travel to the GPU box).  Each
# library is written to a temporary file and renamed, so processes that have the old
# one mapped keep running.
#   workloads/libgskgen.so          seeded input generator (shared input module)
#   oracle/liboracle.so             CPU parity oracle (test infrastructure)
#   paper_0812_2769_b200/libgsk.so  the product: sm_100a kernels behind the C-ABI
NVCC ?= /usr/local/cuda/bin/nvcc
HOSTCXX := g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_0812_2769_b200
CU_SRC := $(wildcard $(PKG)/csrc/*.cu)
CU_HDR := $(wildcard $(PKG)/csrc/*.cuh) include/gsk.h

# AC-2: no FMA contraction anywhere on either side.
NVFLAGS := -O3 $(ARCH) -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude \
           -Xptxas -warn-spills
ORCFLAGS := -O2 -mfma -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -std=c++17
GENFLAGS := -O2 -ffp-contract=off -fopenmp -fPIC -shared -std=c++17

all: workloads/libgskgen.so oracle/liboracle.so $(PKG)/libgsk.so

workloads/libgskgen.so: workloads/gen.cpp
	$(HOSTCXX) $(GENFLAGS) -o $@.tmp $< && mv -f $@.tmp $@

oracle/liboracle.so: oracle/oracle.cpp
	$(HOSTCXX) $(ORCFLAGS) -o $@.tmp $< && mv -f $@.tmp $@

# one object per translation unit (make -j compiles them in parallel), then one link
CU_OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(CU_SRC))

build/obj/%.o: $(PKG)/csrc/%.cu $(CU_HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/libgsk.so: $(CU_OBJ)
	$(NVCC) $(ARCH) -shared -o $@.tmp.so $(CU_OBJ) -lcudart && mv -f $@.tmp.so $@

clean:
	rm -f workloads/libgskgen.so oracle/liboracle.so $(PKG)/libgsk.so
	rm -rf build/obj

.PHONY: all clean
