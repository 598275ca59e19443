#!/bin/bash
# dense first/last blocks on side streams beside the predictor (short prompts): full GPU
# suite on the new library, then A/B (alternated) on 1B, Qwen3 and 8B at 4K tokens
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t8.log 2>&1; tail -3 gpurun_out/t8.log
for i in 1 2; do
  tools/ab_cfg.sh "--config 1b" build/libffwd_noov.so build/libffwd_new.so
  tools/ab_cfg.sh "--config qwen8b --layers 8" build/libffwd_noov.so build/libffwd_new.so
  tools/ab_cfg.sh "--layers 8 --tokens 4096" build/libffwd_noov.so build/libffwd_new.so
done > gpurun_out/ab_overlap.txt 2>&1
cat gpurun_out/ab_overlap.txt
