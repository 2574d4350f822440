# Build of the B200-native DreamDDP engine (no cmake needed).
#
#   paper_2502_11058_b200/lib/libdsx.so        sm_100a kernels + the dsx C-ABI (include/dsx.h)
#   paper_2502_11058_b200/lib/libdreamsched.so the drop-in dreamsched:: C++ API (include/dreamsched)
#   build/parity_tool                          tests/native/parity_tool.cpp against the above
#   build/acceptance                           the reference's acceptance binary compiled
#                                              against this library (drop-in proof; needs
#                                              /root/reference, so only built where present)
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     ?= g++
PKG     := paper_2502_11058_b200
LIB     := $(PKG)/lib
SRC     := $(PKG)/csrc
REF     ?= /root/reference/proj
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -fmad=false -Xptxas -v -Xcompiler -fPIC -Iinclude
CXXFLAGS:= -std=c++20 -O2 -ffp-contract=off -fPIC -Iinclude -Wall -Wextra
# NCCL: link the same libnccl.so.2 torch loads (the venv's nvidia-nccl wheel),
# so one process never mixes two NCCL builds under one soname.
NCCL_LIBDIR ?= $(shell python3 -c "import nvidia,os;print(os.path.join(list(nvidia.__path__)[0],'nccl','lib'))" 2>/dev/null)
NCCL_LINK := $(if $(wildcard $(NCCL_LIBDIR)/libnccl.so.2),-L$(NCCL_LIBDIR) -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_LIBDIR),-lnccl)
HOST_SRCS := $(wildcard $(SRC)/host/*.cpp)
CUDA_SRCS := $(wildcard $(SRC)/cuda/*.cu)
CUDA_HDRS := $(wildcard $(SRC)/cuda/*.cuh)
API_HDRS  := $(wildcard include/dreamsched/*.hpp) include/dsx.h

.PHONY: all clean acceptance
all: $(LIB)/libdsx.so $(LIB)/libdreamsched.so build/parity_tool $(if $(wildcard $(REF)),acceptance build/unit_tests)

# one object per .cu so `make -j` compiles them in parallel; ptxas -v output
# per object in build/ptxas_<name>.log
CUDA_OBJS := $(patsubst $(SRC)/cuda/%.cu,build/obj/%.o,$(CUDA_SRCS))
build/obj/%.o: $(SRC)/cuda/%.cu
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -MMD -MP -c -o $@ $< 2> build/ptxas_$*.log || (cat build/ptxas_$*.log; false)
-include $(CUDA_OBJS:.o=.d)

$(LIB)/libdsx.so: $(CUDA_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(CUDA_OBJS) $(NCCL_LINK)

$(LIB)/libdreamsched.so: $(HOST_SRCS) $(API_HDRS) $(LIB)/libdsx.so
	$(CXX) $(CXXFLAGS) -shared -o $@ $(HOST_SRCS) -L$(LIB) -ldsx -Wl,-rpath,'$$ORIGIN'

build/parity_tool: tests/native/parity_tool.cpp $(LIB)/libdreamsched.so
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Iinclude $< -L$(LIB) -ldreamsched -ldsx \
	    -Wl,-rpath,'$$ORIGIN/../$(LIB)' -o $@

acceptance: build/acceptance
build/acceptance: $(REF)/tests/acceptance/acceptance_main.cpp tests/native/eager_init.cpp $(LIB)/libdreamsched.so
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Iinclude -I$(REF)/tests/support $< tests/native/eager_init.cpp -L$(LIB) -ldreamsched -ldsx \
	    -Wl,-rpath,'$$ORIGIN/../$(LIB)' -o $@

# The reference's own unit suite (proj/tests/unit/*.cpp, doctest) compiled
# unchanged against this library through tests/native/doctest_shim; the
# trainer cases run on the GPU path (tests/test_unit_suite.py).
UNIT_SRCS := $(wildcard $(REF)/tests/unit/*.cpp)
# simulator_test.cpp reads trace JSON with nlohmann/json (the local 3.11.3 header)
JSON_DIR ?= $(shell python3 -c "import os,site;c=[os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages()];print(next((x for x in c if os.path.exists(os.path.join(x,'json.hpp'))),''))")
build/unit_tests: $(UNIT_SRCS) tests/native/doctest_shim/doctest.h $(LIB)/libdreamsched.so
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Iinclude -I$(REF)/tests/support -Itests/native/doctest_shim -I$(JSON_DIR) \
	    -DDREAMSCHED_TEST_DATA_DIR='"/root/repo/tests/golden/data"' $(UNIT_SRCS) -L$(LIB) -ldreamsched -ldsx \
	    -Wl,-rpath,'$$ORIGIN/../$(LIB)' -o $@

clean:
	rm -rf $(LIB) build
