timeout 600 python -m pytest tests/test_bench.py -q 2>&1 | tail -4
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 1500 gpurun_out/bench_c1.json
