# Build for the B200-native curve-alignment library (sm_100a only).
#   make            -> product library + harness + oracle (+ reference oracle if /root/reference exists)
#   make lib        -> paper_2501_17779_b200/libcurvalign_cuda.so
NVCC     ?= /usr/local/cuda/bin/nvcc
# Host C++ libraries are loaded into processes (Python, user binaries) that map
# the system libstdc++.so.6: link it dynamically (the image's default $CXX,
# /opt/gcc/bin/g++, would link libstdc++.a, whose separate iostream/locale
# state is unsafe next to the shared one).
CXX      := $(if $(wildcard /usr/bin/g++),/usr/bin/g++,$(CXX))
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG      := paper_2501_17779_b200
CSRC     := $(PKG)/csrc
BUILD    := build
REF      ?= /root/reference

KERNEL_HDRS := $(wildcard $(CSRC)/*.cuh) $(CSRC)/kernels.h $(CSRC)/fused.h $(CSRC)/largen.h $(CSRC)/elastic.h include/curvalign_cuda.h

.PHONY: all lib synth dropin dropin_test oracle ref clean prof

# Phase-timing build (tools/phase_timing.py): separate .so, never shipped.
prof: $(PKG)/libcurvalign_cuda_prof.so
$(PKG)/libcurvalign_cuda_prof.so: $(CSRC)/fused.cu $(CSRC)/capi.cpp $(CSRC)/kernels.cu $(CSRC)/allpairs.cu $(CSRC)/largen.cu $(CSRC)/dropin_kernels.cu $(CSRC)/gfft.cu $(CSRC)/elastic.cu $(KERNEL_HDRS) $(CSRC)/prof.cuh
	@mkdir -p $(BUILD)/prof
	$(NVCC) $(NVFLAGS) -DCVA_PHASE_TIMING -c $(CSRC)/fused.cu -o $(BUILD)/prof/fused.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/kernels.cu -o $(BUILD)/prof/kernels.o
	$(NVCC) $(NVFLAGS) -x cu -c $(CSRC)/capi.cpp -o $(BUILD)/prof/capi.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/probe.cu -o $(BUILD)/prof/probe.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/allpairs.cu -o $(BUILD)/prof/allpairs.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/largen.cu -o $(BUILD)/prof/largen.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/dropin_kernels.cu -o $(BUILD)/prof/dropin_kernels.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/gfft.cu -o $(BUILD)/prof/gfft.o
	$(NVCC) $(NVFLAGS) -c $(CSRC)/elastic.cu -o $(BUILD)/prof/elastic.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(BUILD)/prof/*.o
all: lib synth dropin dropin_test oracle ref

lib: $(PKG)/libcurvalign_cuda.so
synth: $(PKG)/libcurvalign_synth.so
dropin: $(PKG)/libcurvalign.so

$(BUILD)/kernels.o: $(CSRC)/kernels.cu $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_kernels.log || (cat $(BUILD)/ptxas_kernels.log; exit 1)

$(BUILD)/fused.o: $(CSRC)/fused.cu $(KERNEL_HDRS) $(CSRC)/fused.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_fused.log || (cat $(BUILD)/ptxas_fused.log; exit 1)

$(BUILD)/allpairs.o: $(CSRC)/allpairs.cu $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_allpairs.log || (cat $(BUILD)/ptxas_allpairs.log; exit 1)

$(BUILD)/largen.o: $(CSRC)/largen.cu $(KERNEL_HDRS) $(CSRC)/largen.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_largen.log || (cat $(BUILD)/ptxas_largen.log; exit 1)

$(BUILD)/elastic.o: $(CSRC)/elastic.cu $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_elastic.log || (cat $(BUILD)/ptxas_elastic.log; exit 1)

$(BUILD)/dropin_kernels.o: $(CSRC)/dropin_kernels.cu $(KERNEL_HDRS) $(CSRC)/gfft.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/gfft.o: $(CSRC)/gfft.cu $(CSRC)/gfft.h $(KERNEL_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/capi.o: $(CSRC)/capi.cpp $(CSRC)/kernels.h $(CSRC)/fused.h $(CSRC)/elastic.h include/curvalign_cuda.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(BUILD)/probe.o: $(CSRC)/probe.cu include/curvalign_cuda.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libcurvalign_cuda.so: $(BUILD)/kernels.o $(BUILD)/fused.o $(BUILD)/allpairs.o $(BUILD)/largen.o $(BUILD)/elastic.o $(BUILD)/dropin_kernels.o $(BUILD)/gfft.o $(BUILD)/capi.o $(BUILD)/probe.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^

# Synthetic workload generators (bench harness; host only).
$(PKG)/libcurvalign_synth.so: $(CSRC)/synth.cpp
	$(CXX) -O2 -std=c++20 -fPIC -shared -Wall -o $@ $< -lpthread

# C++ drop-in for the reference API (namespace curvalign), on top of the C ABI.
DROPIN_SRCS := $(wildcard $(CSRC)/dropin/*.cpp)
$(PKG)/libcurvalign.so: $(DROPIN_SRCS) $(wildcard include/curvalign/*.hpp) $(CSRC)/dropin/status.hpp $(PKG)/libcurvalign_cuda.so
	$(CXX) -O2 -std=c++20 -fPIC -shared -Wall -Iinclude -o $@ $(DROPIN_SRCS) \
	    -L$(PKG) -lcurvalign_cuda -Wl,-rpath,'$$ORIGIN'

# C++ tests of the drop-in API (restating the reference's doctest cases); run
# on a GPU by tests/test_gpu_dropin_cpp.py.
tests/cpp/bin/test_dropin: tests/cpp/test_dropin.cpp $(PKG)/libcurvalign.so
	@mkdir -p tests/cpp/bin
	$(CXX) -O2 -std=c++20 -Wall -pthread -Iinclude -o $@ $< -L$(PKG) -lcurvalign -lcurvalign_cuda \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'
dropin_test: tests/cpp/bin/test_dropin

oracle:
	$(MAKE) -C oracle oracle

ref:
	@if [ -d $(REF)/proj/src ]; then $(MAKE) -C oracle ref REF=$(REF); else echo "reference sources absent: using prebuilt oracle/_ref if present"; fi

clean:
	rm -rf $(BUILD) $(PKG)/*.so
	$(MAKE) -C oracle clean
