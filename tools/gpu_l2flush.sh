for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/flush_$c.json 2> gpurun_out/flush_$c.err
  python -c "import json; d=json.load(open('gpurun_out/flush_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), 'ms', d['config']['l2'], d['roofline']['bound'], round(d['roofline']['frac'],3))" || tail -5 gpurun_out/flush_$c.err
done
timeout 300 python -m pytest tests/test_bench.py -q 2>&1 | tail -2
