#!/bin/bash
# On the GPU box: tools/exprun.sh P CONFIG NAME... -> parity check + bench line per variant
P=$1; CFG=$2; shift 2
for n in "$@"; do
  export DGX_LIB=_exp/$n/libdgx.so
  timeout 300 python tools/expcheck.py $P > gpurun_out/exp_$n.check 2>&1; tail -1 gpurun_out/exp_$n.check
  timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/exp_${n}_$CFG.json 2> gpurun_out/exp_${n}_$CFG.err
  python -c "
import json; d=json.load(open('gpurun_out/exp_${n}_$CFG.json')); r=d['roofline']
print('$n $CFG', '%.3f GDoF/s'%(d['value']/1e9), 'frac %.3f'%r['frac'], 'ms %.3f'%d['ms_per_step'])" || tail -3 gpurun_out/exp_${n}_$CFG.err
done
