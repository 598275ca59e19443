#!/bin/bash
# softmax fused into the pooling pass for short prompts: parity + 1B A/B + 1B bench line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py tests/test_gpu_reference_suite.py tests/test_gpu_prefill.py -q -m gpu -x > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
for i in 1 2 3; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_base.so build/libffwd_new.so
done > gpurun_out/ab_softmax.txt 2>&1
cat gpurun_out/ab_softmax.txt
python bench.py --config 1b > gpurun_out/b1_fused.json 2> gpurun_out/b1_fused.err
tail -c 300 gpurun_out/b1_fused.json
