# femforge-b200 build: one in-tree shared library with the C ABI
# (include/femforge_b200.h), the C++ host API (symbolic / fem / codegen /
# meshgen) and the offline-compiled sm_100a kernels; the element kernel itself
# is compiled at run time by NVRTC.
#
#   make            -> paper_1802_03433_b200/libfemforge_b200.so + C++ test binaries
#   make oracle     -> oracle/liboracle.so (+ oracle/_ref when /root/reference exists)
CUDA     ?= /usr/local/cuda
CXX      := g++
NVCC     := $(CUDA)/bin/nvcc
PKG      := paper_1802_03433_b200
SRC      := $(PKG)/csrc
BUILD    := build
ARCH     := -gencode arch=compute_100a,code=sm_100a
INC      := -I$(SRC)/include -Iinclude -I$(CUDA)/include
CXXFLAGS := -std=c++20 -O2 -g -fPIC -Wall -Wextra $(INC)
NVFLAGS  := $(ARCH) -lineinfo -O3 -std=c++17 -Xcompiler -fPIC $(INC)
LDLIBS   := -L$(CUDA)/lib64 -lcudart_static -lrt -ldl -lpthread -Wl,-rpath,$(CUDA)/lib64

CPP_SRCS := $(SRC)/symbolic/symbolic.cpp $(SRC)/fem/fem.cpp $(SRC)/meshgen/meshgen.cpp \
            $(SRC)/codegen/lower.cpp $(SRC)/codegen/element_plan.cpp $(SRC)/codegen/emit.cpp \
            $(SRC)/runtime/nvrtc.cpp $(SRC)/capi/capi.cpp $(SRC)/api/femforge.cpp
CU_SRCS  := $(SRC)/kernels/pattern.cu $(SRC)/kernels/linalg.cu $(SRC)/kernels/validate.cu
OBJS     := $(patsubst $(SRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS)) $(patsubst $(SRC)/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS))
LIB      := $(PKG)/libfemforge_b200.so
ARCHIVE  := $(BUILD)/libfemforge_b200.a

TEST_SRCS := $(wildcard tests/cpp/test_*.cpp)
TEST_BINS := $(patsubst tests/cpp/%.cpp,$(BUILD)/tests/%,$(TEST_SRCS))

all: $(LIB) $(ARCHIVE) $(TEST_BINS)

$(BUILD)/%.o: $(SRC)/%.cpp $(wildcard $(SRC)/include/femforge/*.hpp) include/femforge_b200.h $(SRC)/runtime/runtime.hpp $(SRC)/kernels/assemble_template.inc
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/%.cu.o: $(SRC)/%.cu $(SRC)/kernels/kernels.hpp
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# the shared library exports the C ABI only (ff_*; exports.map)
$(LIB): $(OBJS) $(SRC)/capi/exports.map
	$(CXX) -shared -o $@ $(OBJS) -Wl,--version-script=$(SRC)/capi/exports.map $(LDLIBS)

$(ARCHIVE): $(OBJS)
	@mkdir -p $(dir $@)
	rm -f $@ && ar rcs $@ $(OBJS)

# C++ host-API suites link the static archive (the C++ API is not exported
# by the shared library)
$(BUILD)/tests/%: tests/cpp/%.cpp tests/cpp/check.hpp $(ARCHIVE)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -Itests/cpp $< -o $@ $(ARCHIVE) $(LDLIBS)

oracle:
	$(MAKE) -C oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all oracle clean
