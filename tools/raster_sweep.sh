#!/bin/bash
# Sweep the L2 raster group sizes on the 8B stack (8 layers, short bench).
for r in "$@"; do
  python bench.py --steps 4 --warmup 2 --layers 8 --skip-cpu --skip-dense --raster $r 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_layer']
print('raster $r: %.3f ms/layer  up %.3f down %.3f' % (d['value'], k['up_proj'], k['down_proj']))"
done
