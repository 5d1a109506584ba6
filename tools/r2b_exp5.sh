#!/bin/bash
# tensor-product kernel v3 (staged coalesced neighbour cells, bank-spreading line permutations): parity + benches + ncu
mkdir -p gpurun_out
python -m pytest tests/test_gpu.py tests/test_fullsize.py tests/test_loopback.py -x -q -k "cart or tensor or c1 or c2 or c5 or golden or fp32" > gpurun_out/x5_pytest_cart.log 2>&1; echo pytest_cart_rc=$?; tail -3 gpurun_out/x5_pytest_cart.log
for c in c5 c5f32 c1 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x5_$c.json 2>gpurun_out/x5_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x5_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
ncu --set full --import-source on --clock-control none -k regex:'sipg_cart' -c 1 -o gpurun_out/x5_ncu_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x5_ncu_c5.log 2>&1; echo ncu_c5_rc=$?
for r in gpurun_out/x5_ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details > $b.txt 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
  rm -f $r
done
