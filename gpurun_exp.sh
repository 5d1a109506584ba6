for e in base NO_GEO NO_FACE; do
  if [ $e = base ]; then unset DGX_LIB; else export DGX_LIB=$PWD/exp/$e/libdgx.so; fi
  for c in c4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_${e}_$c.json 2>gpurun_out/exp_${e}_$c.err; python -c "
import json; d=json.load(open('gpurun_out/exp_${e}_$c.json')); print('$e $c', '%.3f GDoF/s'%(d['value']/1e9), 'ms %.3f'%d['ms_per_step'])"; done
done
unset DGX_LIB
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
