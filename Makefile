# Top-level build. Everything is built IN-TREE so the .so files travel to the GPU
# box with gpurun (they are git-ignored, not gpurun-ignored).
#   paper_1606_04884_b200/lib/libpt_b200.so   CUDA kernels + C ABI (include/pt_b200.h)
#   paper_1606_04884_b200/lib/libportten.so   C++ operator API (include/portten/*.hpp)
#   tests/cpp/portten_tests                   C++ test driver (host logic; --gpu parity)
#   oracle/liboracle.so, oracle/_ref/...      TEST-ONLY checkers (oracle/Makefile)
#   integration/_ref/libportten_refdev.so     TEST-ONLY: the reference's backend layer with
#                                             the B200 plug-in in its device slot
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := g++
PKG      := paper_1606_04884_b200
LIBDIR   := $(PKG)/lib
CUDA_INC := /usr/local/cuda/include
CUDA_LIB := /usr/local/cuda/lib64
GENCODE  := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++17 -O3 $(GENCODE) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
            --expt-relaxed-constexpr -Iinclude
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(CUDA_INC)

CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
CU_HDRS  := $(wildcard $(PKG)/csrc/*.cuh) include/pt_b200.h
CU_OBJS  := $(patsubst $(PKG)/csrc/%.cu,build/cu/%.o,$(CU_SRCS))
# host-only parts of the library (the apply-expression compiler)
CC_SRCS  := $(wildcard $(PKG)/csrc/*.cpp)
CC_OBJS  := $(patsubst $(PKG)/csrc/%.cpp,build/cc/%.o,$(CC_SRCS))
HOST_SRCS := $(wildcard $(PKG)/host/*.cpp)
HOST_HDRS := $(wildcard include/portten/*.hpp) include/pt_b200.h

.PHONY: all lib host tests oracle clean
all: lib oracle $(if $(HOST_SRCS),host tests)

lib: $(LIBDIR)/libpt_b200.so
host: $(LIBDIR)/libportten.so
tests: tests/cpp/portten_tests
oracle: lib
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; else echo "oracle: /root/reference absent, keeping prebuilt _ref"; fi
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C integration; else echo "integration: /root/reference absent, keeping prebuilt _ref"; fi

build/cu/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build/cu
	$(NVCC) $(NVFLAGS) -dc -o $@ $<

build/cc/%.o: $(PKG)/csrc/%.cpp include/pt_b200.h
	@mkdir -p build/cc
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(LIBDIR)/libpt_b200.so: $(CU_OBJS) $(CC_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(GENCODE) -shared -Xcompiler -fPIC -o $@ $(CU_OBJS) $(CC_OBJS) -L$(CUDA_LIB) -lcudart_static -ldl -lpthread -lrt

$(LIBDIR)/libportten.so: $(HOST_SRCS) $(HOST_HDRS) $(LIBDIR)/libpt_b200.so
	@mkdir -p $(LIBDIR)
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRCS) -L$(LIBDIR) -lpt_b200 -lnccl -Wl,-rpath,'$$ORIGIN'

# test driver: links the product libraries and, as the checker only, the oracle
tests/cpp/portten_tests: tests/cpp/portten_tests.cpp $(LIBDIR)/libportten.so oracle/oracle.h oracle
	$(CXX) $(CXXFLAGS) -o $@ tests/cpp/portten_tests.cpp -L$(LIBDIR) -lportten -lpt_b200 \
	    -Loracle -loracle -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -Wl,-rpath,'$$ORIGIN/../../oracle' -ldl

clean:
	rm -rf build $(LIBDIR) tests/cpp/portten_tests
	$(MAKE) -C oracle clean
	$(MAKE) -C integration clean
