#!/bin/bash
# top-k with two barriers per radix pass and one (gt, eq) scan: parity, A/B vs HEAD, ncu
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_gpu_sp.py tests/test_gpu_reference_suite.py -q -m gpu -x > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
for i in 1 2; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_base.so build/libffwd_new.so
  tools/ab_cfg.sh "--layers 8" build/libffwd_base.so build/libffwd_new.so
done > gpurun_out/ab_topk2.txt 2>&1
cat gpurun_out/ab_topk2.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:topk_kernel -s 2 -c 1 \
  -o gpurun_out/r2_topk_2bar -f python tools/prof_step.py 8b 1 3 > gpurun_out/ncu_topk2.log 2>&1
tail -n 2 gpurun_out/ncu_topk2.log
