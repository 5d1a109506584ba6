#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/x16_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/x16_pytest.log
for c in c3 c3h; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/x16_$c.json 2>gpurun_out/x16_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x16_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
timeout 300 python bench.py --config sweep --degree 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x16_sweep_p4.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/x16_sweep_p4.json')); print('sweep p4', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
for n in sp7base sp7nc5; do
  DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config sweep --degree 6 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x16_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/x16_$n.json')); print('$n', round(d['ms_per_step'],3))"
done
