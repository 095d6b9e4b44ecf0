# Builds the sm_100a C-ABI library and the test-only C oracle helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -rdc=true -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2510_23649_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/liblrqk_b200.so
# development build with the per-block timeline trace compiled in
# (tools/step_timeline.py loads it through LRQK_LIB_PATH)
TOBJ := $(patsubst $(PKG)/csrc/%.cu,build/trace/%.o,$(SRC))
TLIB := $(PKG)/liblrqk_b200_trace.so
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/lrqk_b200.h

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DLRQK_NO_TRACE -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/trace/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/trace
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/trace/$*.ptxas.log || (cat build/trace/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -rdc=true -shared -o $@ $(OBJ) -lcudart_static -lrt -ldl -lpthread

$(TLIB): $(TOBJ)
	$(NVCC) $(ARCH) -rdc=true -shared -o $@ $(TOBJ) -lcudart_static -lrt -ldl -lpthread

trace: $(TLIB)

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/lrqk.sass

clean:
	rm -rf build $(LIB) $(TLIB)

.PHONY: all trace clean sass
