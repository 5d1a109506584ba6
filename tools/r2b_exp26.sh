#!/bin/bash
mkdir -p gpurun_out
for n in ch7base ch7new ch7new4 ch7base; do
  DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config c5h --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x26_$n.json 2>gpurun_out/x26_$n.err
  python -c "import json; d=json.load(open('gpurun_out/x26_$n.json')); print('$n', round(d['ms_per_step'],3))" || tail -2 gpurun_out/x26_$n.err
done
