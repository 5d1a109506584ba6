#!/bin/bash
# On the GPU box: bench lines + ncu launch list + ncu --set full captures of
# the apply kernel for the configurations given (default: c4 c4h c4g4).
# Each ncu command runs only after the same command has exited 0 without ncu.
TAG=${TAG:-pairs}
for c in ${CONFIGS:-c4 c4h c4g4}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err || { echo "bench $c failed"; continue; }
  ncu --set full --import-source on --clock-control none -k regex:'sipg_(pairs|apply)' -c 1 \
    -o gpurun_out/ncu_full_${c}_$TAG python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_full_${c}_$TAG.log 2>&1
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c4_$TAG.log 2>&1
ls gpurun_out
# reports -> text/csv summaries on the box (gpurun brings back <= 64 MiB)
for r in gpurun_out/ncu_full_*_$TAG.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details > $b.txt 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
  [ "${KEEP_REP:-c4}" != "$(basename $b | sed "s/ncu_full_//; s/_$TAG//")" ] && rm -f $r
done
du -sh gpurun_out
