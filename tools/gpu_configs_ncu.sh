# On the GPU box: gpu tests, C3/C4/C5/C1 bench lines, one ncu --set full capture of the C4 apply kernel
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in c3 c4 c5 c1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', '%.3f GDoF/s'%(d['value']/1e9), 'frac %.3f'%d['roofline']['frac'], 'ms %.3f'%d['ms_per_step'])"; done
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sipg -s 3 -c 1 -o gpurun_out/prof_c4_v2 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
