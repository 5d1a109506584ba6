#!/bin/bash
# tensor-product Cartesian kernel: parity (new tests + every Cartesian case of the suite) and C5/C1/C2 benches against the collocation CART kernels
mkdir -p gpurun_out
python -m pytest tests/test_gpu.py -x -q -k "cart or tensor" > gpurun_out/x2_pytest_cart.log 2>&1; echo pytest_cart_rc=$?; tail -5 gpurun_out/x2_pytest_cart.log
python -m pytest tests -m gpu -x -q > gpurun_out/x2_pytest.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/x2_pytest.log
for c in c5 c5f32 c1 c2; do
  for nt in 0 1; do
    if [ $nt = 1 ]; then export DGX_NO_TENSOR=1; else unset DGX_NO_TENSOR; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x2_$c$nt.json 2>gpurun_out/x2_$c$nt.err
    python -c "import json; d=json.load(open('gpurun_out/x2_$c$nt.json')); print('$c notensor=$nt', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
  done
done
unset DGX_NO_TENSOR
