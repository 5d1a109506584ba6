#!/bin/bash
# C4 ablations (resident face data / no face barriers: timing only) + FWDTRACE parity and timing; C5 CART ncu
DGX_LIB=_exp/fwdtr/libdgx.so timeout 300 python tools/expcheck.py 5 > gpurun_out/e4_fwdtr.check 2>&1; tail -1 gpurun_out/e4_fwdtr.check
bash tools/exppair.sh c4 base fres 1
bash tools/exppair.sh c4 fnosync fwdtr 1
bash tools/exppair.sh c4 base fwdtr 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sipg_apply -c 1 -o gpurun_out/ncu_c5cart python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e4_ncu_c5.log 2>&1; echo ncu_rc=$?
