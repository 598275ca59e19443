#!/bin/bash
# K3 with the gathered W_down rows by cp.async (LSU) instead of TMA gather4: parity on the
# variant library, A/B against the default, ncu of the variant's K3
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
FFWD_LIB=build/libffwd_bldg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -q -m gpu -x > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
for i in 1 2; do
  tools/ab_cfg.sh "--layers 8" build/libffwd_base.so build/libffwd_bldg.so
  tools/ab_cfg.sh "--config 1b" build/libffwd_base.so build/libffwd_bldg.so
done > gpurun_out/ab_k3ldgsts.txt 2>&1
cat gpurun_out/ab_k3ldgsts.txt
FFWD_LIB=build/libffwd_bldg.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:down_proj -s 2 -c 1 \
  -o gpurun_out/r2_k3_ldgsts -f python tools/prof_step.py 8b 1 3 > gpurun_out/ncu_k3l.log 2>&1
tail -n 2 gpurun_out/ncu_k3l.log
