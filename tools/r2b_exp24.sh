#!/bin/bash
mkdir -p gpurun_out
for t in 4 8 16 32; do
  DGX_TILE_Y=$t timeout 300 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x24_c3_t$t.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/x24_c3_t$t.json')); print('c3 tile_y=$t', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
for t in 4 8 16; do
  DGX_TILE_Y=$t timeout 300 python bench.py --config sweep --degree 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x24_p3_t$t.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/x24_p3_t$t.json')); print('sweep p3 tile_y=$t', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
