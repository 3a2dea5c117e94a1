# Build of the B200 ACS library (sm_100a) and the CPU oracle.
#
#   make            -> paper_1605_02669_b200/libacs_b200.so, oracle/liboracle.so
#                      (+ oracle/_ref/libacsref.so when /root/reference exists)
#   make tools      -> build/acs-bench (C++ CLI over the drop-in API)
#
# Built artefacts stay in-tree (git-ignored, not gpurun-ignored) so they travel
# to the GPU box with the snapshot.

NVCC ?= /usr/local/cuda/bin/nvcc
CXX := /usr/bin/g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_1605_02669_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/libacs_b200.so

NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -warn-spills \
           --expt-relaxed-constexpr
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -ffp-contract=off -I include \
            -I /usr/local/cuda/include

CU_SRCS := $(SRC)/k_setup.cu $(SRC)/k_colony.cu $(SRC)/k_micro.cu $(SRC)/capi.cu
CXX_SRCS := $(SRC)/instance.cpp $(SRC)/solver.cpp $(SRC)/stats.cpp
CU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS))
CXX_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CXX_SRCS))
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard include/*.h) $(wildcard include/acs/*.hpp)

all: $(LIB) oracle

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CXX_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lz -ldl

oracle:
	$(MAKE) -s -C oracle

tools: build/acs-bench

build/acs-bench: tools/acs_bench.cpp $(LIB) $(HDRS)
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(PKG) -lacs_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle tools clean

# A/B kernel experiments: make ab V=<name> DEFS="-DFOO=1" builds
# paper_1605_02669_b200/libacs_b200_<name>.so (select with ACS_LIB_VARIANT=<name>);
# COLONY=<file> builds another k_colony.cu (e.g. the previous commit's, as _ab_*.cu)
ab:
	@mkdir -p build/obj_$(V)
	$(NVCC) $(NVFLAGS) $(DEFS) -c $(or $(COLONY),$(SRC)/k_colony.cu) -o build/obj_$(V)/k_colony.o
	$(NVCC) $(NVFLAGS) $(DEFS) -c $(SRC)/k_setup.cu -o build/obj_$(V)/k_setup.o
	$(NVCC) $(NVFLAGS) $(DEFS) -c $(SRC)/capi.cu -o build/obj_$(V)/capi.o
	$(NVCC) $(NVFLAGS) $(DEFS) -c $(SRC)/k_micro.cu -o build/obj_$(V)/k_micro.o
	$(NVCC) $(ARCH) -shared -o $(PKG)/libacs_b200_$(V).so build/obj_$(V)/k_colony.o build/obj_$(V)/k_setup.o \
	  build/obj_$(V)/k_micro.o build/obj_$(V)/capi.o $(CXX_OBJS) -lz -ldl

.PHONY: ab
