#!/bin/bash
# pooling pass: 16 tokens in flight per lane (2 CTAs/SM) vs 8 (3 CTAs/SM), 1B and 8B stacks
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_base.so build/libffwd_pb16.so
  tools/ab_cfg.sh "--layers 8" build/libffwd_base.so build/libffwd_pb16.so
  tools/ab_cfg.sh "--config qwen8b --layers 8" build/libffwd_base.so build/libffwd_pb16.so
done > gpurun_out/ab_pool.txt 2>&1
cat gpurun_out/ab_pool.txt
