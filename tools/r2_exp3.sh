#!/bin/bash
python -m pytest tests/test_fullsize.py -x -q -k "cart or c5" > gpurun_out/e3_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e3_pytest.log
for c in c5 c5f32 c1 c2; do
  for nc in 0 1; do
    if [ $nc = 1 ]; then export DGX_NO_CART=1; else unset DGX_NO_CART; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/e3_$c$nc.json 2>gpurun_out/e3_$c$nc.err
    python -c "import json; d=json.load(open('gpurun_out/e3_$c$nc.json')); print('$c nocart=$nc', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
  done
done
unset DGX_NO_CART
