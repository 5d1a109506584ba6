#!/bin/bash
# CART kernels: parity (gpu tests) + C5/C1 benches; C4 CTA-size sweep
python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_loopback.py -x -q > gpurun_out/e2_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/e2_pytest.log
for c in c5 c5f32; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/e2_$c.json 2>gpurun_out/e2_$c.err
  python -c "import json; d=json.load(open('gpurun_out/e2_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],3), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
for n in c1base c1cart; do
  DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config c1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/e2_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2_$n.json')); print('$n', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step']*1e3,2), 'us')"
done
bash tools/exppair.sh c4 base nc2 1
bash tools/exppair.sh c4 nc3 nc4 1
