# Builds the in-tree CUDA library (sm_100a) that the Python drop-in loads.
#   make -j16            -> paper_2401_10068_b200/libcavi.so
NVCC ?= /usr/local/cuda/bin/nvcc
PY_SITE ?= $(shell python -c 'import sysconfig; print(sysconfig.get_paths()["purelib"])')
NCCL_HOME ?= $(PY_SITE)/nvidia/nccl
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 $(ARCH) -lineinfo -std=c++17 $(EXTRA) -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -I$(NCCL_HOME)/include
PKG := paper_2401_10068_b200
CSRC := $(PKG)/csrc
BUILD ?= build/obj
HDR := $(wildcard $(CSRC)/*.cuh) $(CSRC)/pow5_table.inc include/cavi.h
DIMS := 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15
PASS_OBJS := $(foreach d,$(DIMS),$(BUILD)/pass_d$(d).o)
LIB ?= $(PKG)/libcavi.so

all: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/pass_d%.o: $(CSRC)/pass_inst.cu $(HDR) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DCAVI_D=$* -c -o $@ $<

$(BUILD)/cavi.o: $(CSRC)/cavi.cu $(HDR) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(BUILD)/csv_host.o: $(CSRC)/csv_host.cpp $(CSRC)/numparse.cuh $(CSRC)/pow5_table.inc include/cavi.h | $(BUILD)
	$(CXX) -O3 -std=c++17 -fPIC -Wall -pthread -c -o $@ $<

$(BUILD)/kde.o: $(CSRC)/kde.cu include/cavi.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(BUILD)/cavi.o $(BUILD)/csv_host.o $(BUILD)/kde.o $(PASS_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_HOME)/lib -Xcompiler -pthread

ptxas: | $(BUILD)
	$(NVCC) $(NVFLAGS) -DCAVI_D=3 -Xptxas -v -c -o $(BUILD)/ptxas_d3.o $(CSRC)/pass_inst.cu

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean ptxas
