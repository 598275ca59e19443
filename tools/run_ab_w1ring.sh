#!/bin/bash
# W1 cluster split-K with a 4-deep chunk ring for 32-row tiles: parity + 1B A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -q -m gpu -x > gpurun_out/t12.log 2>&1; tail -2 gpurun_out/t12.log
for i in 1 2 3; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_head.so build/libffwd_new.so
done > gpurun_out/ab_w1ring.txt 2>&1
cat gpurun_out/ab_w1ring.txt
