#!/bin/bash
# ncu --set full: C5 tensor-product kernel, C4 pair kernel (base) and its cell-integral-only ablation (nofsmall)
mkdir -p gpurun_out
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x4_c5.json 2>gpurun_out/x4_c5.err; python -c "import json; d=json.load(open('gpurun_out/x4_c5.json')); print('c5', round(d['value']/1e9,2), round(d['ms_per_step'],3))"
ncu --set full --import-source on --clock-control none -k regex:'sipg_cart' -c 1 -o gpurun_out/x4_ncu_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x4_ncu_c5.log 2>&1; echo ncu_c5_rc=$?
for n in base nofsmall; do
  DGX_LIB=_exp/$n/libdgx.so ncu --set full --import-source on --clock-control none -k regex:'sipg_pairs' -c 1 -o gpurun_out/x4_ncu_$n python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x4_ncu_$n.log 2>&1; echo ncu_${n}_rc=$?
done
for r in gpurun_out/x4_ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details > $b.txt 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
  rm -f $r
done
du -sh gpurun_out
