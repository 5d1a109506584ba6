#!/bin/bash
# HEAD validation (all GPU tests, default bench) + C4 ablations: occupancy (padded smem -> 2 CTAs/SM),
# cell integral alone at 3 / 4 / 5+ CTAs per SM, resident face data, no face barriers, forward traces
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
( time python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/x1_pytest.log 2>&1; echo pytest_rc=$?; tail -16 gpurun_out/x1_pytest.log
timeout 600 python bench.py > gpurun_out/x1_bench_default.json 2> gpurun_out/x1_bench_default.err; echo bench_rc=$?; cat gpurun_out/x1_bench_default.json
for n in base pad2 nofbig nofsmall nofsmall5 fres fnosync fwdtr; do
  DGX_LIB=_exp/$n/libdgx.so timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x1_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/x1_$n.json')); print('$n', round(d['ms_per_step'],3))"
done
