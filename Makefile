# Builds the C-ABI shared library of the B200-native R-distance hot path.
# sm_100a only (B200). No fast-math: the kernels rely on IEEE division,
# sqrt and log.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $(EXTRA)
BUILD ?= build
SRC_DIR := paper_2308_07403_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,$(BUILD)/%.o,$(SRCS))
HDRS := $(wildcard $(SRC_DIR)/*.cuh) include/rdist_b200.h
LIB ?= paper_2308_07403_b200/librdist_b200.so

all: $(LIB)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
