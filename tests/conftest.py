import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("basics"))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


class Case:
    """A golden fixture decoded into its configuration."""

    def __init__(self, name):
        self.name = name
        self.g = load_golden(name)
        meta = self.g["meta"]
        self.d = d = int(meta[0])
        self.cells = [int(c) for c in meta[1:1 + d]]
        self.p = int(meta[1 + d])
        self.periodic = bool(meta[2 + d])
        self.m = int(meta[3 + d])
        self.n_ranks = int(meta[4 + d])
        self.vertex = "eps" in self.g
        self.eps = float(self.g["eps"]) if self.vertex else 0.0
        self.coefficient = bool(self.g["coefficient"]) if self.vertex else False
        self.amplitude = 0.0 if self.vertex else float(self.g["amplitude"])
        # BasisKind: 0 lagrange_gauss_lobatto, 1 lagrange_gauss, 2 hermite_like
        self.basis = int(self.g.get("basis", 0))
        self.basis_name = ("lagrange_gauss_lobatto", "lagrange_gauss", "hermite_like")[self.basis]
        adv = self.g.get("advection")
        self.kind = "advection" if adv is not None else "laplacian"
        self.velocity = tuple(float(v) for v in adv[:3]) if adv is not None else (1.0, 1.0, 1.0)
        self.velocity_field = int(adv[3]) if adv is not None else 0
        self.seeds = sorted(int(k[1:]) for k in self.g if k.startswith("x") and k[1:].isdigit())

    @property
    def cartesian(self):
        return not self.vertex and self.amplitude == 0.0

    def deform(self):
        if self.vertex:
            return ("vertex", self.eps)
        if self.amplitude == 0.0:
            return None
        return ("reference", self.amplitude, self.m)


def rel_linf(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
