# traversal tile height (DGX_TILE_Y) on the single-pencil configurations C3 / C5
for c in c3 c5; do
  for t in 4 8 16 32; do
    DGX_TILE_Y=$t timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/tile_${c}_$t.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/tile_${c}_$t.json')); print('$c tile_y=$t', round(d['ms_per_step'],3))"
  done
done
