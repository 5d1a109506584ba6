#!/bin/bash
# tensor-product kernel: fp32 without staging; full GPU suite; default bench
mkdir -p gpurun_out
for c in c5f32 c5 c1 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/x6_$c.json 2>gpurun_out/x6_$c.err
  python -c "import json; d=json.load(open('gpurun_out/x6_$c.json')); print('$c', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3))"
done
python -m pytest tests -m gpu -x -q > gpurun_out/x6_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/x6_pytest.log
python tools/overlap_timeline.py 2 64 > gpurun_out/x6_overlap_R2.txt 2> gpurun_out/x6_overlap_R2.err; echo overlap_rc=$?; tail -8 gpurun_out/x6_overlap_R2.txt
