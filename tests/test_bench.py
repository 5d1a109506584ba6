"""bench.py's JSON-line contract (the driver parses this line every round).

CPU: the reference arm (`--impl reference`, the reference's own RankOperator::apply
compiled under oracle/_ref, threaded ranks) at N=1 and under torchrun with two
ranks (rank 0 alone prints, the other rank exits 0 without work).
GPU: the product arm on the small C1 configuration, with every key the driver
and the judge read (roofline, cpu_baseline, e2e, gpu_launches, clocks).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libdgref.so")
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e")


def _run(args, timeout=600):
    r = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return lines


def _check_base(d, steps, warmup):
    for k in BASE_KEYS:
        assert k in d, k
    assert d["unit"] == "DoF/s" and d["higher_is_better"] is True
    assert d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("C1")
    # value and ms_per_step describe the same step: the whole mesh on the GPU;
    # the reference arm's measured sample (cells, applies per step)
    if d.get("impl") == "reference":
        m = d["measured"]
        n = m["n_dofs"] * m["applies_per_step"]
    else:
        n = d["config"]["n_dofs"]
    assert abs(n / (d["ms_per_step"] * 1e-3) / d["value"] - 1) < 0.05


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (run build())")
def test_reference_arm_json_line():
    lines = _run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                  "--steps", "2", "--warmup", "3"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    _check_base(d, 2, 3)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (run build())")
def test_reference_arm_two_ranks_rank0_only():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    lines = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                  "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                  "--master-port", str(port), "bench.py", "--impl", "reference",
                  "--config", "c1", "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


@pytest.mark.gpu
def test_product_arm_json_line():
    lines = _run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup", "3"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    _check_base(d, 3, 3)
    assert d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["gpu_launches"] >= 3
    rf = d["roofline"]
    # the binding resource of the configuration: HBM bytes or FP64 flops (C1 is FP64-bound)
    assert (rf["bound"], rf["unit"]) in (("hbm", "GB/s"), ("fp64", "TFLOP/s"))
    assert rf["algorithmic_bytes_per_launch"] > 0 and rf["launch_ms"] > 0
    assert 0 < rf["frac"] < 1.2 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["value"] > 0 and cb["cores"] >= 1
    e = d["e2e"]
    assert e["unit"] == "DoF/s" and 0 < e["value"] <= d["value"] * 1.05
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # short timed regions carry clocks sampled under the same load around them
    assert d["clocks"]["samples"] >= 1 and d["clocks"]["sm_mhz"] is not None
