# Builds the sm_100a extension in-tree (the .so travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude
PKG := paper_2602_00397_b200
SRC := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cpp)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h include/*.h)
LIB := $(PKG)/libffwd_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

clean:
	rm -f $(LIB)

.PHONY: all clean
