# Builds libfemgpu.so in-tree for sm_100a (host C++ runtime + C-ABI; kernels are
# specialised per form at runtime with NVRTC for sm_100a) and the test oracle.
CUDA ?= /usr/local/cuda
NVCC ?= $(CUDA)/bin/nvcc
PKG := paper_2506_17471_b200
SRC := $(PKG)/csrc
OBJDIR := build/obj
LIB := $(PKG)/_lib/libfemgpu.so
CXXSRC := $(SRC)/api.cpp $(SRC)/instance.cpp $(SRC)/emit.cpp $(SRC)/emit_dmma.cpp $(SRC)/jit.cpp $(SRC)/mesh.cpp $(SRC)/tune.cpp $(SRC)/io.cpp $(SRC)/pipeline.cpp $(SRC)/fuse.cpp $(SRC)/reorder.cpp
CUSRC := $(wildcard $(SRC)/*.cu)
HDRS := include/femgpu.h $(SRC)/femgpu_internal.hpp
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr
OBJS := $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CXXSRC)) $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.cu.o,$(CUSRC))

all: $(LIB) oracle adapter

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(OBJDIR)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS) $(SRC)/femgpu.map
	@mkdir -p $(dir $@)
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a -o $@ $(OBJS) -lnvrtc -cudart static -Xlinker -rpath,$(CUDA)/lib64 \
	  -Xlinker --version-script=$(SRC)/femgpu.map -Xlinker --exclude-libs,ALL

oracle:
	$(MAKE) -s -C oracle

# C++ drop-in test (needs the reference headers; skipped with a message when absent)
adapter: $(LIB)
	$(MAKE) -s -C tests/cpp

clean:
	rm -rf build $(LIB)

.PHONY: all oracle adapter clean
