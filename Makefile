# Builds paper_2507_00394_b200/libhx.so (sm_100a) and the oracle's C pieces.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# Every n-th packed pair of forward softmax exponentials on the FMA pipe (0 = all
# on MUFU).  Measured in the GPT-1.3B/32k bench step with the speculative-exp
# forward: 16 (6% of the exps) 4.16-4.17 ms per forward vs 4.25-4.27 with 0 and
# 4.30 with 8; alone, 4 was 4.7% slower.
HX_POLY_EVERY ?= 16
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude -DHX_POLY_EVERY=$(HX_POLY_EVERY)
SRC := $(wildcard paper_2507_00394_b200/csrc/*.cu)
HDR := $(wildcard paper_2507_00394_b200/csrc/*.cuh paper_2507_00394_b200/csrc/*.h include/*.h)
OBJ := $(patsubst paper_2507_00394_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2507_00394_b200/libhx.so

all: $(LIB)

build/%.o: paper_2507_00394_b200/csrc/%.cu $(HDR) Makefile
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared $(OBJ) -o $@

ptxas: $(SRC)
	@for f in $(SRC); do $(NVCC) $(NVFLAGS) -Xptxas -v -c $$f -o /dev/null 2>&1 | grep -E "Function properties|registers|spill|error" ; done

clean:
	rm -rf build $(LIB)

.PHONY: all clean ptxas
