#!/bin/bash
# On the GPU box: tools/expncu.sh NAME [CONFIG] -> gpurun_out/NAME.ncu-rep (ncu --set full, source counters)
N=$1; CFG=${2:-c4}
DGX_LIB=_exp/$N/libdgx.so ncu --set full --import-source on --clock-control none -k regex:'sipg_(pairs|apply)' -c 1 \
  -o gpurun_out/$N python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$N.log 2>&1
tail -1 gpurun_out/ncu_$N.log
