#!/bin/bash
# 512-thread top-k CTAs for few rows: parity + 1B A/B (three alternated rounds)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_gpu_sp.py tests/test_gpu_tp_sp.py tests/test_gpu_reference_suite.py -q -m gpu -x > gpurun_out/t15.log 2>&1; tail -2 gpurun_out/t15.log
for i in 1 2 3; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_head.so build/libffwd_new.so
done > gpurun_out/ab_topk512.txt 2>&1
cat gpurun_out/ab_topk512.txt
