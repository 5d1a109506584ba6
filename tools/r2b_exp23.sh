#!/bin/bash
mkdir -p gpurun_out
run() { # name args
  DGX_LIB=_exp/$1/libdgx.so timeout 300 python bench.py $2 --steps 15 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x23_$1.json 2>gpurun_out/x23_$1.err
  python -c "import json; d=json.load(open('gpurun_out/x23_$1.json')); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))" || tail -2 gpurun_out/x23_$1.err
}
for n in k6base k6nc3 k6nc3b k6nc2 k6sp k6sp1 k6sp2 k6w1 k6base; do run $n "--config c4"; done
