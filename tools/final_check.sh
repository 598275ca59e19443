# Round-end check on one B200: GPU tests, smoke, the three bench configs, ncu launch list.
set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/b8.json 2> gpurun_out/b8.err
python bench.py --config 1b > gpurun_out/b1.json 2> gpurun_out/b1.err
python bench.py --config qwen8b > gpurun_out/bq.json 2> gpurun_out/bq.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --skip-cpu --skip-dense --skip-ttft > gpurun_out/ncu_bench.log 2>&1
tail -c 300 gpurun_out/b8.json; tail -c 200 gpurun_out/b1.json; tail -c 200 gpurun_out/bq.json
