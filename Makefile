# libhybrid_cuda.so: sm_100a kernels + C ABI (include/hybrid_cuda.h), built in-tree so the
# .so travels to the GPU box with gpurun.  `make oracle` builds the CPU checker (tests only).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v -cudart static
PKG := paper_2005_05371_b200
SRCS := $(PKG)/csrc/tma_host.cu $(PKG)/csrc/amf.cu $(PKG)/csrc/wiener.cu $(PKG)/csrc/small.cu $(PKG)/csrc/stretch.cu $(PKG)/csrc/wstats.cu $(PKG)/csrc/freq.cu $(PKG)/csrc/multi.cu $(PKG)/csrc/capi.cu $(PKG)/csrc/phantom.cpp
HDRS := $(PKG)/csrc/hyb_internal.cuh $(PKG)/csrc/tma.cuh $(PKG)/csrc/networks.cuh $(PKG)/csrc/amf_core.cuh $(PKG)/csrc/w1_core.cuh include/hybrid_cuda.h
LIB := $(PKG)/libhybrid_cuda.so
HOSTLIB := $(PKG)/libdenoise_cuda.so
CXX ?= g++
CPPTEST := tests/cpp/test_host
PGMTEST := tests/cpp/test_pgm

all: $(LIB) $(HOSTLIB) oracle $(CPPTEST) $(PGMTEST)

# C++ host driver with the reference's filter API (paper_2005_05371_b200/host/denoise_cuda.hpp)
$(HOSTLIB): $(PKG)/host/denoise_cuda.cpp $(PKG)/host/pgm_io.cpp $(PKG)/host/denoise_cuda.hpp include/hybrid_cuda.h $(LIB)
	$(CXX) -std=c++20 -O2 -fPIC -Wall -Wextra -shared -o $@ $(PKG)/host/denoise_cuda.cpp $(PKG)/host/pgm_io.cpp -L$(PKG) -lhybrid_cuda -Wl,-rpath,'$$ORIGIN'

# the reference's unit tests re-expressed against the host driver (run by tests/test_cpp_host.py)
$(CPPTEST): tests/cpp/test_host.cpp oracle/hyb_oracle.c $(HOSTLIB)
	$(CXX) -std=c++20 -O2 -Wall -Wextra -o $@ tests/cpp/test_host.cpp -x c oracle/hyb_oracle.c -x none \
		-L$(PKG) -ldenoise_cuda -lhybrid_cuda -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 2> build_ptxas.log || (cat build_ptxas.log; exit 1)
	@grep -E "registers|spill" build_ptxas.log | sed 's/^ptxas info    : //' | head -40

# phase-timestamp build of the same library (tools/trace_amf.py); not used by tests or bench
trace: $(PKG)/libhybrid_cuda_trace.so
$(PKG)/libhybrid_cuda_trace.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -DHYB_TRACE -shared -o $@ $(SRCS) -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 2> /dev/null

# PGM I/O tests (CPU only)
$(PGMTEST): tests/cpp/test_pgm.cpp $(HOSTLIB)
	$(CXX) -std=c++20 -O2 -Wall -Wextra -o $@ tests/cpp/test_pgm.cpp -L$(PKG) -ldenoise_cuda -lhybrid_cuda \
		-Wl,-rpath,'$$ORIGIN/../../$(PKG)'

# A/B variant of the same library (tools/ab.sh): make alt ALTDEF=-DHYB_SMALL_NT=256
ALTDEF ?=
alt: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) $(ALTDEF) -shared -o $(PKG)/libhybrid_cuda_alt.so $(SRCS) -lcufft -Xlinker -rpath,/usr/local/cuda/lib64 2> build_alt.log || (grep -i error build_alt.log; exit 1)

oracle:
	$(MAKE) -C oracle --no-print-directory

clean:
	rm -f $(LIB) $(PKG)/libhybrid_cuda_trace.so $(HOSTLIB) $(CPPTEST) $(PGMTEST) build_ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean trace alt
