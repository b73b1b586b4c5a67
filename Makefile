# Builds the C-ABI engine library for sm_100a and the CPU self-check library.
NVCC ?= nvcc
PKG := paper_2104_10949_b200
CSRC := $(PKG)/csrc
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
HDRS := $(wildcard $(CSRC)/*.cuh) include/mpc3_b200.h
OBJS := build/elementwise.o build/gemm.o build/deal.o build/layers.o
LIB := $(PKG)/libmpc3b200.so
HOSTLIB := $(PKG)/libmpc3hostcheck.so

all: $(LIB) $(HOSTLIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS)

$(HOSTLIB): $(CSRC)/hostcheck.cpp $(HDRS)
	g++ -O2 -std=c++17 -fPIC -shared -Wno-unknown-pragmas -o $@ $(CSRC)/hostcheck.cpp

clean:
	rm -rf build $(LIB) $(HOSTLIB)

.PHONY: all clean
