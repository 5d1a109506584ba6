#!/bin/bash
# full-size parity tests + no-face occupancy ablation (C4)
python -m pytest tests/test_fullsize.py -x -q --durations=20 > gpurun_out/fs.log 2>&1; echo fullsize_rc=$?; tail -25 gpurun_out/fs.log
bash tools/exppair.sh c4 base nofbig 1
bash tools/exppair.sh c4 nofsmall base 1
