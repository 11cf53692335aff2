# Build of the B200 Goldbach verifier (sm_100a).  `make` builds:
#   paper_2603_07850_b200/libgoldbach_b200.so   CUDA kernels + C-ABI + C++ host layer
#   paper_2603_07850_b200/bin/goldbach           the CLI (drop-in for proj/tools/main.cpp)
#   paper_2603_07850_b200/bin/test_host          C++ unit tests of the host layer
#   paper_2603_07850_b200/bin/ref_api_conformance every reference API symbol, exact signatures
#   oracle/liboracle.so                          CPU oracle (test infrastructure)
NVCC ?= nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2603_07850_b200
CSRC := $(PKG)/csrc
BIN := $(PKG)/bin
OBJ := build/obj
CUDA_HOME ?= /usr/local/cuda
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -warn-spills -I$(CSRC) -Iinclude $(NVEXTRA)
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -pthread -I$(CSRC)/include -Iinclude -I$(CUDA_HOME)/include
LIB := $(PKG)/libgoldbach_b200.so

CU_SRCS := $(CSRC)/gb_kernels.cu $(CSRC)/gb_capi.cu
HOST_SRCS := $(wildcard $(CSRC)/host/*.cpp)
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS))
HOST_OBJS := $(patsubst $(CSRC)/host/%.cpp,$(OBJ)/host/%.o,$(HOST_SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h include/*.h $(CSRC)/include/goldbach/*.hpp)

all: $(LIB) cli oracle

$(OBJ)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/host/%.o: $(CSRC)/host/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) -shared $(ARCH) -Xcompiler -fPIC $^ -o $@ -lcudart_static -lrt -lpthread -ldl

cli: $(LIB)
	@if [ -f $(CSRC)/tools/goldbach_main.cpp ]; then mkdir -p $(BIN) && \
	  $(CXX) $(CXXFLAGS) $(CSRC)/tools/goldbach_main.cpp -o $(BIN)/goldbach -L$(PKG) -lgoldbach_b200 -Wl,-rpath,'$$ORIGIN/..' && \
	  $(CXX) $(CXXFLAGS) $(CSRC)/tools/test_host.cpp -o $(BIN)/test_host -L$(PKG) -lgoldbach_b200 -Wl,-rpath,'$$ORIGIN/..' && \
	  $(CXX) $(CXXFLAGS) $(CSRC)/tools/ref_api_conformance.cpp -o $(BIN)/ref_api_conformance -L$(PKG) -lgoldbach_b200 -Wl,-rpath,'$$ORIGIN/..'; fi

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(BIN) oracle/liboracle.so

.PHONY: all cli oracle clean
