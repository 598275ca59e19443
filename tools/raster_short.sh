#!/bin/bash
# raster group sizes (up, down blocks per L2 group) at the short-prompt configs
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2; do
  for r in 32,16 8,8 16,8 16,16 64,32 4,4; do
    echo "## 1b raster $r"; tools/ab_cfg.sh "--config 1b --raster $r" build/libffwd_head.so
  done
  for r in 32,16 16,8 64,32; do
    echo "## qwen8b raster $r"; tools/ab_cfg.sh "--config qwen8b --layers 8 --raster $r" build/libffwd_head.so
  done
done > gpurun_out/raster_short.txt 2>&1
grep -A2 "##" gpurun_out/raster_short.txt | grep -v "^--" | paste - - - | awk '{print $2,$3,$4,$8,$9}'
