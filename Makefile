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
CLI     := $(PKG)/tcsparse-b200

all: lib cli probe oracle

lib: $(LIB)

# The reference CLI (ref tools/tcsparse.cpp) on the B200 library.
cli: $(CLI)

$(CLI): $(PKG)/cli/tcsparse_b200.cpp include/tcs/tcs.h $(LIB)
	g++ -std=c++17 -O2 -Wall -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -ltcsparse_b200 \
	    -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -Wl,-rpath,'$$ORIGIN'

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/tcs_internal.cuh $(wildcard include/tcs/*.h)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -ldl

oracle: lib
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(CLI)
	$(MAKE) -s -C oracle clean

# Hardware L2 -> SM gather ceiling, run by bench.py (roofline.l2_gather).
probe: tools/l2_gather_peak

tools/l2_gather_peak: tools/l2_gather_peak.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<

.PHONY: all lib cli probe oracle clean
