#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/x19_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/x19_pytest.log
for p in 3 4 5 6 7 8; do
  timeout 300 python bench.py --config sweep --degree $p --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x19_sweep_p$p.json 2>gpurun_out/x19_sweep_p$p.err
  python -c "import json; d=json.load(open('gpurun_out/x19_sweep_p$p.json')); print('sweep p$p', d['config']['cells'][0], round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
