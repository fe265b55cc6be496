# Builds the B200-native library and the CPU checkers.
#
#   make            -> paper_2409_16997_b200/lib/libifa_b200.so (sm_100a) + oracle
#   make ref        -> oracle/_ref/* (needs /root/reference; CPU checker only)
#
# Every CUDA source is compiled for exactly one target:
#   -gencode arch=compute_100a,code=sm_100a
# No fast-math: the kernels restate the reference's IEEE float expressions.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2409_16997_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/lib/libifa_b200.so
SRCS := $(CSRC)/abi.cu $(CSRC)/host_abi.cu $(CSRC)/attn.cu $(CSRC)/attn_half.cu $(CSRC)/attn_pp.cu $(CSRC)/attn_ws.cu $(CSRC)/quant.cu $(CSRC)/code_bounds.cpp \
        $(CSRC)/tensor_io.cpp
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/ifa_b200.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

CLI := $(PKG)/lib/ifa_b200

all: $(LIB) $(CLI) oracle

# command-line front end (quantize / info on IFA1 files), C++ over the C-ABI
$(CLI): tools/ifa_b200_cli.cpp include/ifa_b200.h $(LIB)
	g++ -O2 -std=c++17 -Iinclude -o $@ $< -L$(PKG)/lib -lifa_b200 -Wl,-rpath,'$$ORIGIN'

OBJDIR := $(PKG)/lib/obj
OBJS := $(patsubst $(CSRC)/%,$(OBJDIR)/%.o,$(SRCS))

# one object per translation unit, so `make -j` compiles the kernels in parallel
$(OBJDIR)/%.o: $(CSRC)/% $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS) -lcuda
	@cat $(OBJDIR)/*.ptxas.log > $(PKG)/lib/ptxas.log

oracle:
	$(MAKE) -s -C oracle all

ref: $(LIB)
	$(MAKE) -s -C oracle ref refa verify

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(PKG)/lib/sass.txt

clean:
	rm -rf $(PKG)/lib
	$(MAKE) -s -C oracle clean

.PHONY: all oracle ref sass clean
