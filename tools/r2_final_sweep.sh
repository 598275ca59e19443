#!/bin/bash
# final library: GPU suite + smoke, and the configs[4] sweep (sparsity x length, 4-layer stacks)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t6.log 2>&1; tail -3 gpurun_out/t6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke6.log 2>&1; tail -2 gpurun_out/smoke6.log
timeout 1500 python tools/sweep.py > gpurun_out/sweep_final.jsonl 2> gpurun_out/sweep_final.err
wc -l gpurun_out/sweep_final.jsonl
