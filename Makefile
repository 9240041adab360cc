# Builds paper_1903_03237_b200/libfastmnmf.so for sm_100a (B200) with nvcc.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
CSRC := paper_1903_03237_b200/csrc
OBJ := build/obj
LIB := paper_1903_03237_b200/libfastmnmf.so
HDRS := $(wildcard $(CSRC)/*.cuh) include/fastmnmf.h
SRCS := $(CSRC)/fm_api.cu $(CSRC)/fm_f32.cu $(CSRC)/fm_f64.cu $(CSRC)/fm_fused_f32.cu $(CSRC)/fm_fused_f64.cu $(CSRC)/fm_bin.cu
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.o,$(SRCS))

all: $(LIB)

$(OBJ)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
