#!/bin/bash
# On the GPU box: tools/exppair.sh CONFIG A B [ROUNDS] -> alternating bench runs (--steps 30) of two experiment builds
CFG=$1; A=$2; B=$3; R=${4:-2}
for i in $(seq $R); do
  for n in $A $B; do
    DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config $CFG --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pair_$n.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/pair_$n.json')); print('$n', round(d['ms_per_step'],3))"
  done
done
