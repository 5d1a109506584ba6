CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sipg -s 3 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_full.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_full.log
