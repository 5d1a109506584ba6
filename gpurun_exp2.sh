./tools/fp64_pipes
timeout 900 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -2
for c in c4 c3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', '%.3f GDoF/s'%(d['value']/1e9), 'frac %.3f'%d['roofline']['frac'], 'ms %.3f'%d['ms_per_step'])"; done
