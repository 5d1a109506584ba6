#!/bin/bash
# On the GPU box: C2 degree sweep (2D 256^2 Dirichlet, p = 1..10), one bench line per degree
for p in 1 2 3 4 5 6 7 8 9 10; do
  timeout 300 python bench.py --config c2 --degree $p --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    > gpurun_out/c2_p$p.json 2> gpurun_out/c2_p$p.err
  python -c "
import json; d=json.load(open('gpurun_out/c2_p$p.json')); r=d['roofline']
print('p=$p', 'GDoF/s %.2f' % (d['value']/1e9), 'us %.1f' % (d['ms_per_step']*1e3), r['bound'], 'frac %.3f' % r['frac'])" || tail -2 gpurun_out/c2_p$p.err
done
