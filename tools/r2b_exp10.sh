#!/bin/bash
# cart kernel: y-neighbour scalars taken in the y-phase (fewer live registers), staging in both precisions
mkdir -p gpurun_out
python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_loopback.py -x -q -k "cart or tensor or c1 or c2 or c5 or golden or fp32" > gpurun_out/x11_pytest_cart.log 2>&1; echo pytest_cart_rc=$?; tail -3 gpurun_out/x11_pytest_cart.log
for c in c5h c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x11_$c.json 2>gpurun_out/x11_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x11_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
