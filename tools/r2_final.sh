#!/bin/bash
# Round-2 evidence run on one B200: GPU tests, smoke, bench (8B / 1B / Qwen3 / reference),
# ncu launch list of the bench step, and one ncu --set full capture of K2, K3, the norm,
# the pooling pass, the scores GEMM and the top-k (one 8B/16K layer, 3rd launch).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/b8.json 2> gpurun_out/b8.err
python bench.py --config 1b > gpurun_out/b1.json 2> gpurun_out/b1.err
python bench.py --config qwen8b > gpurun_out/bq.json 2> gpurun_out/bq.err
timeout 600 python bench.py --impl reference > gpurun_out/bref.json 2> gpurun_out/bref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --skip-cpu --skip-dense --skip-ttft --skip-f32-pred > gpurun_out/ncu_bench.log 2>&1
for k in up_proj down_proj rmsnorm_ring pooled_kernel gemm_f64_kernel topk_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/r2_$k -f python tools/prof_step.py 8b 1 3 > gpurun_out/ncu_$k.log 2>&1
done
tail -c 300 gpurun_out/b8.json; tail -c 200 gpurun_out/b1.json; tail -c 200 gpurun_out/bq.json; tail -c 200 gpurun_out/bref.json
