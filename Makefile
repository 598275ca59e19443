# Builds the sm_100a extension in-tree (the .so travels to the GPU box with gpurun).
# One object per translation unit, so `make -j` compiles them in parallel.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude
PKG := paper_2602_00397_b200
SRC := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cpp)
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h include/*.h)
OBJDIR := build/obj
OBJ := $(patsubst $(PKG)/csrc/%,$(OBJDIR)/%.o,$(SRC))
LIB := $(PKG)/libffwd_b200.so

all: $(LIB)

$(OBJDIR)/%.o: $(PKG)/csrc/% $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -f $(LIB) $(OBJ)

.PHONY: all clean
