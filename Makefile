# Builds the sm_100a product library in-tree (travels to the GPU box with gpurun)
# and the CPU oracle (test infrastructure, oracle/Makefile).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG  := paper_2605_08523_b200
LIB  := $(PKG)/lib/libfermiforge_b200.so
SRCS := $(PKG)/csrc/ffg_capi.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/fermiforge/ffg.h
NVFLAGS := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc \
           -Xptxas -v --expt-relaxed-constexpr

all: lib oracle

lib: $(LIB)
$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/lib/ptxas.log || (cat $(PKG)/lib/ptxas.log; false)
	@grep -E "registers|spill" $(PKG)/lib/ptxas.log | sed 's/^/  /' | head -20

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB)
.PHONY: all lib oracle clean
