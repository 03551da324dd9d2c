# Builds the in-tree C-ABI library (travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
SRC := paper_2410_01754_b200/csrc
LIB := paper_2410_01754_b200/_lib/liblfmm.so
HDRS := $(wildcard $(SRC)/*.cuh) include/lfmm.h
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -Xptxas -v

all: $(LIB)

$(LIB): $(SRC)/lfmm_api.cu $(HDRS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)/lfmm_api.cu -lcudart 2> $(SRC)/../_lib/ptxas.log || (cat $(SRC)/../_lib/ptxas.log; exit 1)

clean:
	rm -f $(LIB)

.PHONY: all clean

# profiling variant of the M2L kernel (per-CTA wait counters), never shipped
prof: $(SRC)/lfmm_api.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -DLFMM_HM_PROF -shared -o paper_2410_01754_b200/_lib/liblfmm_prof.so $(SRC)/lfmm_api.cu -lcudart 2> /dev/null
