#!/bin/bash
# Round 2: bench contract checks and new bench lines (sweep, c4_64 both arms,
# c5f32 fp32 roofline, short-region clocks, FP32/FP64 pipe peaks)
./tools/fp64_pipes | tee gpurun_out/pipes.txt
python -m pytest tests/test_bench.py -x -q > gpurun_out/bc_testbench.log 2>&1; echo test_bench_rc=$?
for c in c1 c5f32; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bc_$c.json 2> gpurun_out/bc_$c.err; echo $c rc=$?
done
for p in 3 4 5 6 7 8; do
  timeout 300 python bench.py --config sweep --degree $p --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bc_sweep_p$p.json 2> gpurun_out/bc_sweep_p$p.err; echo sweep p=$p rc=$?
done
timeout 600 python bench.py --config c4_64 --steps 20 --warmup 5 --ref-cells 64 > gpurun_out/bc_c4_64.json 2> gpurun_out/bc_c4_64.err; echo c4_64 rc=$?
timeout 900 python bench.py --config c4_64 --impl reference --steps 3 --warmup 3 --ref-cells 64 > gpurun_out/bc_c4_64_ref.json 2> gpurun_out/bc_c4_64_ref.err; echo c4_64 ref rc=$?
for f in gpurun_out/bc_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(sys.argv[1], round(d["value"]/1e9, 3), "GDoF/s", round(d["ms_per_step"], 3), "ms", r.get("bound"), r.get("frac") and round(r["frac"], 3), d.get("clocks"), (d.get("cpu_baseline") or {}).get("value"))
except Exception as e:
    print(sys.argv[1], "parse error", e)
PY
done
