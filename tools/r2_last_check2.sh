#!/bin/bash
# HEAD after the narrow pooling CTAs: GPU suite, smoke, 1B and Qwen3 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t11.log 2>&1; tail -2 gpurun_out/t11.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke11.log 2>&1; tail -1 gpurun_out/smoke11.log
python bench.py --config 1b > gpurun_out/b1_last.json 2> gpurun_out/b1_last.err
python bench.py --config qwen8b > gpurun_out/bq_last.json 2> gpurun_out/bq_last.err
tail -c 200 gpurun_out/b1_last.json; echo; tail -c 200 gpurun_out/bq_last.json
