#!/bin/bash
# NCCL single-rank transport test, torchrun N=1 bench sanity, ncu of the fp32 tensor kernel (C5)
mkdir -p gpurun_out
python -m pytest tests/test_loopback.py -x -q -k "nccl or errors" > gpurun_out/x8_pytest.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/x8_pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --config c1 --no-cpu-baseline > gpurun_out/x8_torchrun1.json 2> gpurun_out/x8_torchrun1.err; echo torchrun_rc=$?; cut -c1-200 gpurun_out/x8_torchrun1.json
ncu --set full --import-source on --clock-control none -k regex:'sipg_cart' -c 1 -o gpurun_out/x8_ncu_c5f32 python bench.py --config c5f32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x8_ncu_c5f32.log 2>&1; echo ncu_rc=$?
for r in gpurun_out/x8_ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details > $b.txt 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  rm -f $r
done
