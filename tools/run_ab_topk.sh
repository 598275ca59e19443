#!/bin/bash
# K1 changes (cluster top-k, h-resident W2 for short prompts, cluster split-K W1):
# parity tests on the new library, A/B (alternated), ncu of the cluster top-k and W1
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -q -m gpu -x > gpurun_out/t2.log 2>&1; tail -3 gpurun_out/t2.log
for i in 1 2; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_base.so build/libffwd_nocl.so build/libffwd_new.so
  tools/ab_cfg.sh "--layers 8" build/libffwd_base.so build/libffwd_nocl.so build/libffwd_new.so
done > gpurun_out/ab_topk.txt 2>&1
cat gpurun_out/ab_topk.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:topk_cluster -s 2 -c 1 \
  -o gpurun_out/r2_topk_cluster -f python tools/prof_step.py 8b 1 3 > gpurun_out/ncu_topk.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_cluster -s 2 -c 1 \
  -o gpurun_out/r2_w1_cluster_1b -f python tools/prof_step.py 1b 1 3 > gpurun_out/ncu_w1.log 2>&1
tail -2 gpurun_out/ncu_topk.log gpurun_out/ncu_w1.log
