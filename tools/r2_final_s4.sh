#!/bin/bash
# Round-2 closing evidence run on one B200 (after the short-prompt predictor GEMMs and the
# two-barrier top-k): GPU suite, smoke, bench lines (8B / 1B / Qwen3 / reference arm), the
# ncu launch list of the bench step, ncu --set full of the changed K1 kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/b8.json 2> gpurun_out/b8.err
python bench.py --config 1b > gpurun_out/b1.json 2> gpurun_out/b1.err
python bench.py --config qwen8b > gpurun_out/bq.json 2> gpurun_out/bq.err
timeout 900 python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --skip-cpu --skip-dense --skip-ttft --skip-f32-pred > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1b.csv \
  python bench.py --config 1b --steps 2 --warmup 1 --skip-cpu --skip-dense --skip-ttft --skip-f32-pred > gpurun_out/ncu_b1.log 2>&1
for k in gemm_f64_cluster gemm_f64_resident topk_kernel pooled_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/r2s4_1b_$k -f python tools/prof_step.py 1b 1 3 > gpurun_out/ncu_1b_$k.log 2>&1
done
tail -c 400 gpurun_out/b8.json; echo; tail -c 300 gpurun_out/b1.json; echo; tail -c 300 gpurun_out/bq.json; echo; tail -c 300 gpurun_out/bref.json
