#!/bin/bash
# Round-2 verification on one GPU box: all GPU tests, smoke(), the default bench line and the
# reference arm, the ncu launch list of the default bench command and one --set full capture
# of its kernel, bench lines of the other BASELINE configurations.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r2f_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r2f_smoke.log
timeout 900 python bench.py > gpurun_out/r2f_bench_c4.json 2> gpurun_out/r2f_bench_c4.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2f_bench_c4_reference.json 2> gpurun_out/r2f_bench_c4_reference.err; echo ref_rc=$?
for c in c3 c5 c5f32 c1 c2 c4h c3h c5h c4_64; do
  timeout 600 python bench.py --config $c > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
for f in gpurun_out/r2f_bench_*.json; do python - "$f" <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print(sys.argv[1].split('r2f_bench_')[1], 'value %.2f GDoF/s'%(d['value']/1e9), 'ms %.4f'%d['ms_per_step'], r.get('bound'), 'frac %.3f'%(r.get('frac') or 0), 'e2e %.2f'%((e.get('value') or 0)/1e9), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))
PY
done
for p in 1 2 3 4 5 6 7 8 9 10; do
  timeout 300 python bench.py --config c2 --degree $p --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2f_c2_p$p.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2f_c2_p$p.json')); print('c2 p=$p', round(d['value']/1e9,2), 'GDoF/s', round(d['ms_per_step']*1e3,1), 'us', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_launches_c4.log 2>&1; echo launches_rc=$?
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:'sipg_cart' -c 1 -o gpurun_out/r2f_ncu_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f_ncu_c5.log 2>&1; echo ncu_rc=$?
for r in gpurun_out/r2f_ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details > $b.txt 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  rm -f $r
done
