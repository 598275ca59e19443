#!/bin/bash
# A/B the library variants in build/ on the 8B layer stack (short bench, 8 layers)
for so in "$@"; do
  echo "== $so"
  FFWD_LIB=$so timeout 300 python bench.py --steps 5 --warmup 3 --layers 8 --skip-cpu --skip-dense --skip-ttft 2>&1 | python -c "
import json,sys
for line in sys.stdin:
    if line.startswith('{'):
        d=json.loads(line); print('ms/layer %.3f' % d['value'], {k: round(v,3) for k,v in d['kernels_ms_per_layer'].items()})
    else: print(line.rstrip()[:200])
"
done
