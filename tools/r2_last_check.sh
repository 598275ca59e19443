#!/bin/bash
# last check of the committed HEAD build: GPU suite, smoke, 8B bench line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t9.log 2>&1; tail -2 gpurun_out/t9.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke9.log 2>&1; tail -1 gpurun_out/smoke9.log
python bench.py > gpurun_out/b8_last.json 2> gpurun_out/b8_last.err; tail -c 250 gpurun_out/b8_last.json
