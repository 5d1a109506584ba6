#!/bin/bash
# One-call GPU check used during development: parity tests, then a bench
# line per configuration (device-timed apply).
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-c4 c3 c5 c1 c2}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
print('$c', '%.3f GDoF/s'%(d['value']/1e9), 'frac %.3f'%r['frac'], 'ms %.3f'%d['ms_per_step'], 'B/DoF %.1f'%r['bytes_per_dof'])" || tail -3 gpurun_out/bench_$c.err
done
