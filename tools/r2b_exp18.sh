#!/bin/bash
# CTA shapes of the pair kernel: k=4 (sweep p=3), k=6 (C4), k=8 (sweep p=7)
mkdir -p gpurun_out
run() { # name degree/config
  DGX_LIB=_exp/$1/libdgx.so timeout 300 python bench.py $2 --steps 15 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x18_$1.json 2>gpurun_out/x18_$1.err
  python -c "import json; d=json.load(open('gpurun_out/x18_$1.json')); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))" || tail -2 gpurun_out/x18_$1.err
}
for n in k4base k4nc4 k4nc8 k4nc16 k4base; do run $n "--config sweep --degree 3"; done
for n in base k6nc7 base; do run $n "--config c4"; done
for n in k8base k8nc1 k8nc3 k8base; do run $n "--config sweep --degree 7"; done
