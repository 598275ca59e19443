#!/bin/bash
# Build a compile-time variant of the library: tools/build_variant.sh NAME "-DFLAG=V ..."
# -> build/libffwd_NAME.so (load it with FFWD_LIB=build/libffwd_NAME.so; tools/ab.sh).
set -e
cd "$(dirname "$0")/.."
mkdir -p build
PKG=paper_2602_00397_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude $2 -shared \
  -o build/libffwd_$1.so $PKG/csrc/*.cu $PKG/csrc/*.cpp
echo build/libffwd_$1.so
