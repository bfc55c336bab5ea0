# Build of the B200-native library (sm_100a only) and the CPU oracle.
#   make            -> paper_2412_11007_b200/libtcsparse_b200.so + oracle/
#   make lib        -> the CUDA library only
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Iinclude \
           --expt-relaxed-constexpr -Xptxas -warn-spills
PKG     := paper_2412_11007_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
LIB     := $(PKG)/libtcsparse_b200.so

all: lib oracle

lib: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/tcs_internal.cuh include/tcs/tcs.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all lib oracle clean
