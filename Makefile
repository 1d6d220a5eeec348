# Build of the product library (paper_2401_16543_b200/libkfvm_b200.so) and the
# CPU oracle (oracle/libkfvm_oracle.so, test infrastructure only).
#
# The CUDA translation unit is compiled for sm_100a only, with -fmad=false:
# every FP64 fused multiply-add in the kernels is written explicitly, so the
# device arithmetic is the pinned FP contract shared with the oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -std=gnu++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra
MINB ?= 2
MMAMINB ?= 3
EXTRA ?=
NVFLAGS := $(ARCH) $(EXTRA) -DKFVM_FAST_MINB=$(MINB) -DKFVM_MMA_MINB=$(MMAMINB) -std=c++17 -O3 -lineinfo -fmad=false -Xcompiler -fPIC,-ffp-contract=off \
           -Xptxas -v --expt-relaxed-constexpr

PKG := paper_2401_16543_b200
SRC := $(PKG)/csrc
LIB := $(PKG)/libkfvm_b200.so
ORACLE := oracle/libkfvm_oracle.so
BUILD := build

all: $(LIB) $(ORACLE)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/kfvm_table.o: $(SRC)/kfvm_table.cpp include/kfvm_b200.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/kfvm_ic.o: $(SRC)/kfvm_ic.cpp $(SRC)/kfvm_ic_eval.h $(SRC)/kfvm_ic_host.h include/kfvm_b200.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(SRC)/kfvm_gen.cuh: tools/gen_kernels.py
	python tools/gen_kernels.py

$(BUILD)/kfvm_gpu.o: $(SRC)/kfvm_gpu.cu $(SRC)/kfvm_gen.cuh $(SRC)/kfvm_device.cuh $(SRC)/kfvm_recon.cuh $(SRC)/kfvm_recon_u.cuh $(SRC)/kfvm_ic_eval.h include/kfvm_b200.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_kfvm_gpu.txt || (cat $(BUILD)/ptxas_kfvm_gpu.txt; false)

$(LIB): $(BUILD)/kfvm_table.o $(BUILD)/kfvm_ic.o $(BUILD)/kfvm_gpu.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lquadmath -ldl

$(ORACLE): oracle/kfvm_oracle.cpp oracle/kfvm_oracle.h include/kfvm_b200.h
	$(CXX) $(CXXFLAGS) -O3 -march=x86-64-v2 -shared $< -o $@ -lpthread

clean:
	rm -rf $(BUILD) $(LIB) $(ORACLE)

.PHONY: all clean
