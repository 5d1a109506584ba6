#!/bin/bash
# tensor-product kernel v2 (all global loads in the prologue): parity + C5/C1/C2 benches, CTAs-per-SM variants at k=7
mkdir -p gpurun_out
python -m pytest tests/test_gpu.py tests/test_fullsize.py -x -q -k "cart or tensor or c1 or c2 or c5" > gpurun_out/x3_pytest_cart.log 2>&1; echo pytest_cart_rc=$?; tail -3 gpurun_out/x3_pytest_cart.log
for c in c5 c5f32 c1 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x3_$c.json 2>gpurun_out/x3_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x3_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
for n in t7base t7mb4 t7mb5; do
  DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x3_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/x3_$n.json')); print('$n', round(d['ms_per_step'],3))"
done
