"""Quick parity check of a kernel-experiment build (tools/expbuild.sh) on
3D configurations of one degree, against the C restatement oracle.
Usage: DGX_LIB=_exp/NAME/libdgx.so python tools/expcheck.py P"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import test_gpu as T  # noqa: E402

p = int(sys.argv[1])
cfgs = [
    (3, [3, 3, 2], p, False, ("reference", 0.04, 2), False, 1),
    (3, [3, 2, 3], p, True, ("reference", 0.04, 2), False, 1),
    (3, [3, 3, 4], p, False, ("vertex", 0.1), True, 2),
    (3, [4, 3, 3], p, True, None, False, 3),
    (3, [3, 3, 2], p, False, ("reference", 0.04, 2), False, 2, "hermite_like"),
    (3, [3, 2, 2], p, True, ("vertex", 0.1), False, 1, "lagrange_gauss"),
    # brick-aligned meshes (every face of a brick CTA internal or external)
    (3, [4, 4, 4], p, True, ("reference", 0.04, 2), False, 1),
    (3, [4, 4, 2], p, False, ("vertex", 0.1), True, 2),
    (3, [2, 2, 2], p, True, None, False, 1),
    (3, [4, 2, 4], p, False, ("reference", 0.04, 2), False, 1, "hermite_like"),
]
bad = 0
for c in cfgs:
    try:
        T.run_random_config(torch, c)
        print("ok  ", T._cfg_id(c))
    except AssertionError as e:
        bad += 1
        print("FAIL", T._cfg_id(c), e)
print("expcheck", "FAILED" if bad else "passed", os.environ.get("DGX_LIB"))
sys.exit(1 if bad else 0)
