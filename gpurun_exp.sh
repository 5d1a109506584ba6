for e in base NO_NBR NO_FGEO NO_LINE NO_GEO NO_FACE; do
  if [ $e = base ]; then unset DGX_LIB; else export DGX_LIB=$PWD/exp/$e/libdgx.so; fi
  timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_${e}.json 2>gpurun_out/exp_${e}.err; python -c "
import json; d=json.load(open('gpurun_out/exp_${e}.json')); print('$e', '%.3f GDoF/s'%(d['value']/1e9), 'ms %.3f'%d['ms_per_step'])"
done
