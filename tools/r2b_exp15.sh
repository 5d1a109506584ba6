#!/bin/bash
# C3 (k=5) CTA shapes of the single-pencil kernel; decomposition overhead on one GPU
mkdir -p gpurun_out
bash tools/exppair.sh c3 sp5base sp5nc6 1
bash tools/exppair.sh c3 sp5nc5 sp5nc5b4 1
bash tools/exppair.sh c3 sp5nc4 sp5base 1
timeout 1500 python tools/decomposition_overhead.py 128 5 1 2 4 8 > gpurun_out/x15_decomp.txt 2> gpurun_out/x15_decomp.err; echo decomp_rc=$?; cat gpurun_out/x15_decomp.txt; tail -3 gpurun_out/x15_decomp.err
