# Build of the B200-native WSM path (sm_100a only) and its CPU checkers.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $(EXTRA)
CSRC      := paper_1011_0093_b200/csrc
LIB       := paper_1011_0093_b200/lib/libcolorq_b200.so
SHIM_TEST := build/shim_test
CLI       := build/colorq_b200
IO_TEST   := build/io_test

all: $(LIB) oracle $(SHIM_TEST) $(CLI) $(IO_TEST)

$(LIB): $(CSRC)/capi.cu $(CSRC)/common.cuh $(CSRC)/hist.cuh $(CSRC)/points.cuh $(CSRC)/wsm.cuh $(CSRC)/map.cuh $(CSRC)/prep.cuh include/colorq_b200.h
	mkdir -p $(dir $@) build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC)/capi.cu 2> build/ptxas.log || (cat build/ptxas.log; false)

# C++ drop-in shim test (tests/cpp/shim_test.cpp), linked against the CUDA library.
$(SHIM_TEST): tests/cpp/shim_test.cpp include/colorq_b200/colorq.hpp include/colorq_b200.h $(LIB)
	mkdir -p build
	g++ -O2 -std=c++20 -Iinclude -o $@ tests/cpp/shim_test.cpp -L$(dir $(LIB)) -lcolorq_b200 \
	    -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))'

# The reference CLI's quantize command on the library (tools/colorq_b200_cli.cpp).
$(CLI): tools/colorq_b200_cli.cpp include/colorq_b200/colorq.hpp include/colorq_b200/io.hpp include/colorq_b200/bench.hpp include/colorq_b200.h $(LIB)
	mkdir -p build
	g++ -O2 -std=c++20 -Iinclude -o $@ tools/colorq_b200_cli.cpp -L$(dir $(LIB)) -lcolorq_b200 \
	    -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))'

# Host-only PPM / palette codec driver (tests/test_io_cpu.py; no GPU needed).
$(IO_TEST): tests/cpp/io_test.cpp include/colorq_b200/colorq.hpp include/colorq_b200/io.hpp $(LIB)
	mkdir -p build
	g++ -O2 -std=c++20 -Iinclude -o $@ tests/cpp/io_test.cpp -L$(dir $(LIB)) -lcolorq_b200 \
	    -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))'

oracle:
	$(MAKE) -s -f oracle/Makefile

clean:
	rm -rf build paper_1011_0093_b200/lib oracle/build

.PHONY: all oracle clean
