# Top-level build: the product library (sm_100a only) and the CPU oracle.
#   paper_2602_02846_b200/lib/libkinoplan_b200.so   C-ABI + kernels (the product)
#   oracle/build/libkpo.so, oracle/_ref/ref_kat      test infrastructure
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
PKG = paper_2602_02846_b200
CSRC = $(PKG)/csrc
LIB = $(PKG)/lib/libkinoplan_b200.so
CLI = $(PKG)/bin/kinoplan
# --fmad=false: only explicit fmaf() fuses (the pinned fp32 recipe)
NVFLAGS = $(ARCH) -std=c++17 -O3 -lineinfo --fmad=false -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v
HDRS = $(CSRC)/kp_types.h $(CSRC)/kp_math.cuh include/kinoplan_b200.h

all: $(LIB) $(CLI) oracle

$(CSRC)/kp_kernels.o: $(CSRC)/kp_kernels.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/ptxas_kernels.log || (cat $(CSRC)/ptxas_kernels.log; false)

$(CSRC)/kp_capi.o: $(CSRC)/kp_capi.cpp $(HDRS)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(CSRC)/kinoplan.o: $(CSRC)/kinoplan.cpp include/kinoplan_b200/kinoplan.hpp include/kinoplan_b200.h
	g++ -std=c++20 -O2 -fPIC -ffp-contract=off -Iinclude -c $< -o $@

$(CSRC)/bench.o: $(CSRC)/bench.cpp include/kinoplan_b200/bench.hpp include/kinoplan_b200/kinoplan.hpp
	g++ -std=c++20 -O2 -fPIC -ffp-contract=off -Iinclude -c $< -o $@

$(CSRC)/kinoplan_host.o: $(CSRC)/kinoplan_host.cpp include/kinoplan_b200/kinoplan.hpp
	g++ -std=c++20 -O2 -fPIC -ffp-contract=off -Iinclude -c $< -o $@

$(LIB): $(CSRC)/kp_kernels.o $(CSRC)/kp_capi.o $(CSRC)/kinoplan.o $(CSRC)/bench.o $(CSRC)/kinoplan_host.o
	mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -lrt -lpthread -ldl

# The `kinoplan plan|bench|validate|report` command line.
$(CLI): $(CSRC)/kinoplan_cli.cpp $(LIB) include/kinoplan_b200/bench.hpp
	mkdir -p $(PKG)/bin
	g++ -std=c++20 -O2 -Iinclude $< -o $@ -L$(PKG)/lib -lkinoplan_b200 -Wl,-rpath,'$$ORIGIN/../lib'

oracle:
	$(MAKE) -C oracle

# Product library with the device invariant checks compiled in (KP_ASSERT in
# kp_types.h): same path and name, so the GPU tests run against it unchanged.
checks:
	$(MAKE) -B $(LIB) NVFLAGS="$(NVFLAGS) -DKP_CHECKS"


clean:
	rm -f $(CSRC)/*.o $(LIB) $(CLI)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean checks
