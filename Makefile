# Build for the refsig B200 path. `make` builds everything that does not need
# the reference checkout; `make ref` additionally builds oracle/_ref from
# /root/reference (only present in the dev container).
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -Xptxas -v $(NVEXTRA)
CPUFLAGS := -O3 -std=c++20 -fPIC -march=x86-64-v3 -ffp-contract=off -pthread
REF_INC  ?= /root/reference/proj/include

PKG   := paper_1810_03099_b200
CSRC  := $(PKG)/csrc
LIBDIR:= $(PKG)/lib
BUILD := build

CU_SRCS := $(CSRC)/k0_text.cu $(CSRC)/k1_count.cu $(CSRC)/scan.cu $(CSRC)/k2_sign.cu $(CSRC)/k3_pairs.cu $(CSRC)/k3_tc.cu \
           $(CSRC)/k4_simhash.cu $(CSRC)/k5_exact.cu $(CSRC)/k5_tc.cu $(CSRC)/k6_formats.cu $(CSRC)/capi.cu
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HDRS    := $(CSRC)/common.cuh $(CSRC)/kernels.cuh $(CSRC)/tc_common.cuh include/refsig_gpu.h

GPU_LIB := $(LIBDIR)/librefsig_gpu.so
GEN_LIB := $(LIBDIR)/libmrcgen.so
ORC_LIB := oracle/liboracle.so
REF_LIB := oracle/_ref/librefshim.so
CPP_CHK := $(LIBDIR)/refsig_gpu_cpp_check

all: $(GPU_LIB) $(GEN_LIB) $(ORC_LIB) $(CPP_CHK) tools

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(GPU_LIB): $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared $(CU_OBJS) -o $@ -lcudart

$(GEN_LIB): $(CSRC)/gen/corpus_gen.cpp include/mrcgen.h
	@mkdir -p $(LIBDIR)
	$(CXX) $(CPUFLAGS) -shared -Iinclude $< -o $@

$(ORC_LIB): oracle/oracle.cpp oracle/oracle.h
	$(CXX) $(CPUFLAGS) -shared -Ioracle $< -o $@

$(CPP_CHK): tests/cpp/gpu_api_check.cpp include/refsig/gpu.hpp include/refsig_gpu.h $(GPU_LIB)
	$(CXX) -O2 -std=c++20 -Iinclude $< -o $@ -L$(LIBDIR) -lrefsig_gpu -Wl,-rpath,'$$ORIGIN'

ref: $(REF_LIB)

$(REF_LIB): oracle/ref_shim.cpp
	@mkdir -p oracle/_ref
	$(CXX) $(CPUFLAGS) -shared -I$(REF_INC) $< -o $@

clean:
	rm -rf $(BUILD) $(LIBDIR)/*.so $(CPP_CHK) $(ORC_LIB) $(REF_LIB)

.PHONY: all ref clean

TOOLS := tools/alu_peaks
tools: $(TOOLS)
tools/alu_peaks: tools/alu_peaks.cu
	$(NVCC) -O3 -std=c++17 $(ARCH) -lineinfo --extended-lambda $< -o $@
.PHONY: tools
