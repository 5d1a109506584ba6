#!/bin/bash
mkdir -p gpurun_out
bash tools/exppair.sh c3 sp5cur sp5nc1 1
bash tools/exppair.sh c3 sp5nc1b sp5cur 1
