#!/bin/bash
# Round-2 baseline on the GPU box: gpu tests + bench lines of c4/c3/c5/c5f32
python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest_rc=$? 
for c in c4 c3 c5 c5f32; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2b_$c.json 2> gpurun_out/r2b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/r2b_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],3), 'ms', d['roofline']['bound'], round(d['roofline']['frac'],3), d['clocks'])"
done
