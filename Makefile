# Builds the sm_100a C-ABI library and the test-only C oracle helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -rdc=true -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2510_23649_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/liblrqk_b200.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/common.cuh $(PKG)/csrc/select_common.cuh $(PKG)/csrc/mma_common.cuh include/lrqk_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -rdc=true -shared -o $@ $(OBJ) -lcudart_static -lrt -ldl -lpthread

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/lrqk.sass

clean:
	rm -rf build $(LIB)

.PHONY: all clean sass
