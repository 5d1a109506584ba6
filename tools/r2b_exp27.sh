#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/x27_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/x27_pytest.log
for c in c5h c5 c5f32; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x27_$c.json 2>gpurun_out/x27_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x27_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
