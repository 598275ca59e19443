#!/bin/bash
# K3 with 4 producer warps (16 gathered rows each per stage) vs 8: parity on the variant + 8B/1B A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
FFWD_LIB=build/libffwd_p4.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "layer or dense or edge" > gpurun_out/t16.log 2>&1; tail -2 gpurun_out/t16.log
for i in 1 2; do
  tools/ab_cfg.sh "--layers 8" build/libffwd_head.so build/libffwd_p4.so
  tools/ab_cfg.sh "--config 1b" build/libffwd_head.so build/libffwd_p4.so
done > gpurun_out/ab_k3p4.txt 2>&1
cat gpurun_out/ab_k3p4.txt
