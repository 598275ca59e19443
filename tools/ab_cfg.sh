#!/bin/bash
# A/B library variants on one bench config: tools/ab_cfg.sh "BENCH ARGS" LIB...
args="$1"; shift
for so in "$@"; do
  echo "== $so"
  FFWD_LIB=$so timeout 300 python bench.py --steps 5 --warmup 3 $args --skip-cpu --skip-dense --skip-ttft --skip-f32-pred --skip-alt 2>&1 | python -c "
import json,sys
for line in sys.stdin:
    if line.startswith('{'):
        d=json.loads(line); print('ms/layer %.4f' % d['value'], {k: round(v,4) for k,v in d['kernels_ms_per_layer'].items()})
    elif 'rror' in line: print(line.rstrip()[:200])
"
done
