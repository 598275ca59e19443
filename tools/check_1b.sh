#!/bin/bash
# GPU suite + smoke at HEAD, the 1B bench line, and the ncu launch list of the 1B step
# (real per-kernel durations at 32 blocks, where the predictor's fixed cost matters most).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py --config 1b --skip-cpu > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1b.csv \
  python bench.py --config 1b --steps 2 --warmup 1 --skip-cpu --skip-dense --skip-ttft --skip-f32-pred > gpurun_out/ncu_b1.log 2>&1
tail -c 300 gpurun_out/b1.json
