#!/bin/bash
mkdir -p gpurun_out
run() { # name args
  DGX_LIB=_exp/$1/libdgx.so timeout 300 python bench.py $2 --steps 15 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x21_$1.json 2>gpurun_out/x21_$1.err
  python -c "import json; d=json.load(open('gpurun_out/x21_$1.json')); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))" || tail -2 gpurun_out/x21_$1.err
}
for n in sp5nc1b sp5mb22 sp5mb24 sp5nc1b; do run $n "--config c3"; done
for n in sp7base sp7nc1 sp7base; do run $n "--config sweep --degree 6"; done
for n in sp9base sp9nc1 sp9base; do run $n "--config sweep --degree 8"; done
for n in ct7base ct7nc1 ct7nc2 ct7base; do run $n "--config c5"; done
