# libhsx: sm_100a kernels + C ABI of the H-SADMM sync step.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := paper_2512_14628_b200/csrc/hsx_kernels.cu paper_2512_14628_b200/csrc/hsx_abi.cu
HDR := paper_2512_14628_b200/csrc/hsx_kernels.cuh include/hsx.h
LIB := paper_2512_14628_b200/libhsx.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(SRC)

nohints: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DHSX_NO_L2_HINTS -shared -cudart static -o paper_2512_14628_b200/libhsx_nohints.so $(SRC)

cq32: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DHSX_CAND_QUADS=32 -shared -cudart static -o paper_2512_14628_b200/libhsx_cq32.so $(SRC)

trace: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DHSX_TRACE $(TRACE_FLAGS) -shared -cudart static -o paper_2512_14628_b200/libhsx_trace.so $(SRC)

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/hsx_kernels.o paper_2512_14628_b200/csrc/hsx_kernels.cu

clean:
	rm -f $(LIB)

.PHONY: all clean ptxas trace nohints cq32
