#!/bin/bash
# cart kernel with in-CTA x-neighbour sharing: parity + benches; PCIe duplex and default bench (e2e) twice
mkdir -p gpurun_out
python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_loopback.py -x -q -k "cart or tensor or c1 or c2 or c5 or golden or fp32" > gpurun_out/x7_pytest_cart.log 2>&1; echo pytest_cart_rc=$?; tail -3 gpurun_out/x7_pytest_cart.log
for c in c5 c5f32 c1 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x7_$c.json 2>gpurun_out/x7_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x7_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
python tools/pcie_duplex.py
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/x7_default_$i.json 2> gpurun_out/x7_default_$i.err
  python -c "import json; d=json.load(open('gpurun_out/x7_default_$i.json')); print('default', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2))"
done
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.width.current --format=csv
