# Builds the sm_100a search library (C ABI: include/givf_b200.h) in-tree.
NVCC ?= nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-ffp-contract=off \
          --expt-relaxed-constexpr -Xptxas --warn-on-spills
SRC = $(wildcard paper_1802_02422_b200/csrc/*.cu)
HDR = $(wildcard paper_1802_02422_b200/csrc/*.cuh paper_1802_02422_b200/csrc/*.h) include/givf_b200.h
OBJ = $(patsubst paper_1802_02422_b200/csrc/%.cu,build/%.o,$(SRC))
LIB = paper_1802_02422_b200/_lib/libgivf_b200.so

all: $(LIB) oracle

build/%.o: paper_1802_02422_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -lrt -lpthread -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all clean oracle
