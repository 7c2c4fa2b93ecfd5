# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
NVCC    ?= /usr/local/cuda/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v
PKG     := paper_2407_10449_b200
CSRC    := $(PKG)/csrc
SRCS    := $(CSRC)/gemm_f64.cu $(CSRC)/gemm_i8.cu $(CSRC)/latency.cu $(CSRC)/small.cu $(CSRC)/cp.cu $(CSRC)/ess_chain.cu $(CSRC)/aux_kernels.cu $(CSRC)/runtime.cu
OBJS    := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS    := $(CSRC)/common.cuh $(CSRC)/internal.h include/tmvn.h

all: $(PKG)/libtmvn.so oracle/liboracle.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libtmvn.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

oracle/liboracle.so: oracle/oracle.cpp
	g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ $<

clean:
	rm -rf build $(PKG)/libtmvn.so oracle/liboracle.so

.PHONY: all clean

# profiling variant (tools/phase_timing.py), never loaded by the product path
build/timing/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build/timing
	$(NVCC) $(NVFLAGS) -DTMVN_PHASE_TIMING -c $< -o $@ 2> build/timing/$*.log || (cat build/timing/$*.log; false)

build/libtmvn_timing.so: $(patsubst $(CSRC)/%.cu,build/timing/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static

timing: build/libtmvn_timing.so
.PHONY: timing

# A/B variants of the library (tools/ab_time.py): make variant TAG=x VFLAGS="-D..."
build/var_$(TAG)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build/var_$(TAG)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $< -o $@ 2> build/var_$(TAG)/$*.log || (cat build/var_$(TAG)/$*.log; false)

build/libtmvn_$(TAG).so: $(patsubst $(CSRC)/%.cu,build/var_$(TAG)/%.o,$(SRCS))
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static

variant: build/libtmvn_$(TAG).so
.PHONY: variant
