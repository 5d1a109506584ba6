"""Benchmark of the B200 SIPG-Laplacian apply (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config c4|c3|c5|c5f32|c1|c2|c4h|c3h|c5h] [--cells n]

One step = one y = A u over the whole mesh (all ranks). Default workload:
BASELINE.json configs[3] ("C4"): 3D SIPG Laplacian, deformed 128^3-cell hex
mesh (vertex bump x + 0.1 h sin 2pi x sin 2pi y sin 2pi z), p = 5, variable
coefficient a(x) = 1 + 0.5 sin(pi x) cos(pi y) at the quadrature points,
fp64, 452,984,832 DoFs; u ~ U[-1,1] from seed 3 (std::mt19937 convention).
Cells are split in contiguous lexicographic slabs over N GPUs (strong
scaling) with NCCL ghost exchange overlapped with interior cells.

Rank 0 prints ONE JSON line. Timing: W warm-up steps, then K steps
bracketed by barrier + cudaDeviceSynchronize, CUDA events on the launching
stream, max over ranks. Inputs (u 3.6 GB + geometry ~49 GB) exceed the
126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (d, cells, p, periodic, geometry kind, coefficient, precision, seed, label)
    "c4": (3, 128, 5, False, "vertex", True, "fp64", 3,
           "C4: 3D SIPG, deformed 128^3, p=5, a(x) folded, fp64"),
    "c3": (3, 64, 4, False, "vertex", False, "fp64", 2,
           "C3: 3D SIPG, deformed 64^3, p=4, per-q J^-T and JxW, fp64"),
    "c5": (3, 160, 6, False, "cart", False, "fp64", 4,
           "C5: 3D SIPG, Cartesian 160^3, p=6, affine (compressed), fp64"),
    "c5f32": (3, 160, 6, False, "cart", False, "fp32", 4,
              "C5: 3D SIPG, Cartesian 160^3, p=6, affine (compressed), fp32"),
    "c1": (3, 16, 3, True, "cart", False, "fp64", 0,
           "C1: 3D SIPG, periodic Cartesian 16^3, p=3, fp64"),
    "c2": (2, 256, 5, False, "cart", False, "fp64", 1,
           "C2: 2D SIPG, Dirichlet Cartesian 256^2, p=5, fp64"),
    # the same workloads with the reference's default Laplacian basis for
    # p >= 3, Hermite-like (make_operator_config, operators.cpp:27-41)
    "c4h": (3, 128, 5, False, "vertex", True, "fp64", 3,
            "C4h: 3D SIPG, deformed 128^3, p=5, a(x) folded, Hermite-like basis, fp64"),
    "c3h": (3, 64, 4, False, "vertex", False, "fp64", 2,
            "C3h: 3D SIPG, deformed 64^3, p=4, Hermite-like basis, fp64"),
    "c5h": (3, 160, 6, False, "cart", False, "fp64", 4,
            "C5h: 3D SIPG, Cartesian 160^3, p=6, affine, Hermite-like basis, fp64"),
}
# C4 at the paper's Table-4 size (BASELINE.json configs[3]'s "~56.6M DoFs" is
# the 64^3 mesh): the size the reference arm can also run whole on the host
CONFIGS["c4_64"] = (3, 64, 5, False, "vertex", True, "fp64", 3,
                    "C4 at 64^3: 3D SIPG, deformed 64^3, p=5, a(x) folded, fp64 (56.6M DoFs)")
# the BASELINE metric's 3D degree sweep p=3..8 (--degree): BASELINE vertex
# deformation, per-q J^-T and JxW (g3), cells per direction chosen so the
# mesh holds >= 1e8 DoFs (SWEEP_CELLS)
CONFIGS["sweep"] = (3, 0, 5, False, "vertex", False, "fp64", 2,
                    "3D degree sweep: SIPG, deformed n^3 (>= 1e8 DoFs), per-q J^-T and JxW, fp64")
SWEEP_CELLS = {p: int(np.ceil((1e8 / (p + 1) ** 3) ** (1 / 3))) for p in range(1, 11)}
# the paper's other operator on the C4 workload size (reference mesh
# deformation, amplitude 0.05, mapping degree 2; constant transport field)
CONFIGS["a4"] = (3, 128, 5, False, "mesh", False, "fp64", 3,
                 "A4: 3D advection, deformed 128^3 (reference mapping m=2), p=5, c=(0.85,0.6,0.35), fp64")
L2_BYTES = 126 * 1024 ** 2  # B200 L2
FLUSH_BYTES = 512 * 1024 ** 2
ADVECTION = {"a4": (0.85, 0.6, 0.35)}
# the paper's geometry variant G4 (merged coefficient, 6 instead of 10
# doubles per point) on the C3 / C4 workloads
CONFIGS["c4g4"] = CONFIGS["c4"][:8] + ("C4g4: C4 with geometry variant g4 (merged coefficient)",)
CONFIGS["c3g4"] = CONFIGS["c3"][:8] + ("C3g4: C3 with geometry variant g4 (merged coefficient)",)
VARIANT = {"c4g4": "g4", "c3g4": "g4"}
# BasisKind per config (default: the nodal Gauss-Lobatto basis BASELINE names)
BASIS = {"c4h": "hermite_like", "c3h": "hermite_like", "c5h": "hermite_like"}
# reference instrumented flop count per DoF (counters x W / applies,
# bench.cpp:339), SURVEY.md s.8d
# reference counter flops per DoF of C2 (2D, 256^2, Dirichlet) by degree
C2_FLOPS_PER_DOF = {1: 76.00, 2: 74.67, 3: 86.00, 4: 90.24, 5: 100.00, 6: 105.80, 7: 115.00,
                    8: 121.48, 9: 130.40, 10: 137.26}
# 3D reference counter flops per DoF by degree (alpha / k^3 of the reference
# counters, tiled cell path + faces; exact for any mesh)
SWEEP_FLOPS_PER_DOF = {3: 198.0, 4: 215.52, 5: 240.0, 6: 260.82, 7: 285.0, 8: 307.11}
REF_FLOPS_PER_DOF = {"c4": 240.0, "c4_64": 240.0, "c3": 215.52, "c5": 260.82, "c5f32": 260.82,
                     "c1": 198.0, "c2": 105.80,
                     # Hermite-like: plain (not even-odd) S passes, same counters
                     "c4h": 268.0, "c3h": 242.4, "c5h": 293.14, "a4": 93.0,
                     "c4g4": 240.0, "c3g4": 215.52}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak(prec="fp64"):
    """FP64 (DFMA) or FP32 (FFMA) pipe peak measured by tools/fp64_pipes.cu
    (profiles/fp64_peak.json); nominal B200 figures otherwise."""
    key, nominal = ("fp64_dfma_tflops", 37.0) if prec == "fp64" else ("fp32_ffma_tflops", 74.0)
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)[key]), "measured (tools/fp64_pipes.cu)"
    except Exception:
        return nominal, "nominal"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, load=None):
        self.index = index
        self.proc = None
        self.lines = []
        self.bracket = []
        # load(): enqueues (asynchronously) ~0.3 s of the same work, so that
        # a one-shot query just before and just after a short timed region
        # sees the clocks under this load (the 100 ms sampler never fires
        # inside ms-scale regions)
        self.load = load

    def query_under_load(self):
        if self.load is None:
            return
        try:
            self.load()
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=20).stdout
            self.bracket += [ln.strip() for ln in out.splitlines() if ln.strip()]
        except Exception:
            pass

    def __enter__(self):
        self.query_under_load()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.query_under_load()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        during = len(self.lines)
        lines = self.lines if during >= 3 else self.lines + self.bracket
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if during < 3:
            out["window"] = (f"{during} sample(s) inside the timed region + {len(self.bracket)} "
                             "taken under the same load just before and after it")
        return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class RefBench:
    """Reference CPU apply (oracle/_ref/libdgref.so = the unmodified
    reference RankOperator + GhostExchanger over run_ranks threads,
    bench.cpp:128-166) on a bounded sample of the workload: the same
    configuration at a reduced cell count, all host cores as threaded
    ranks, the better lane width of W in {4, 8}."""

    def __init__(self, cfg_name, sample_cells=None, degree=None):
        from oracle import oracle as O
        from oracle import reflib as R
        d, n, p, periodic, kind, coef, prec, seed, label = CONFIGS[cfg_name]
        if degree:
            p = degree
        cores = os.cpu_count() or 1
        if sample_cells is None:
            sample_cells = {3: 16, 2: 128}[d]
        cells = [sample_cells] * d
        self.cells = cells
        self.n_ranks = min(cores, int(np.prod(cells)))
        geo = None
        if kind == "vertex":
            P = O.Problem(d, cells, p, periodic=periodic, deform=("vertex", 0.1),
                          coefficient=coef, n_ranks=1)
            geo = {k: P.geom[k] for k in ("inv_jac_t", "jxw", "face_jxw", "face_jni",
                                          "face_jne", "penalty")}
            geo["compressed"] = False
        best = None
        for W in (4, 8):
            adv = ADVECTION.get(cfg_name)
            w = R.World(d, cells, p, n_ranks=self.n_ranks, periodic=periodic, W=W, geometry=geo,
                        basis=BASIS.get(cfg_name, "lagrange_gauss_lobatto"),
                        amplitude=0.05 if kind == "mesh" else 0.0,
                        mapping_degree=2 if kind == "mesh" else 1,
                        kind="advection" if adv else "laplacian",
                        velocity=adv or (1.0, 1.0, 1.0),
                        variant=VARIANT.get(cfg_name, "g3"))
            w.time(1)
            t = min(w.time(1) for _ in range(3))
            if best is None or t < best[0]:
                best = (t, W, w)
        t1, self.W, self.world = best
        self.n_dofs = self.world.n_dofs
        # applies per timed step: >= 0.5 s of CPU work (run_benchmark times
        # ceil(0.02 s / est) applies per repetition, bench.cpp:309-319)
        self.inner = max(1, int(np.ceil(0.5 / max(t1, 1e-6))))
        self.sample = (f"{label.split(':')[0]} shape (p={p}) at {sample_cells}^{d} cells "
                       f"({self.n_dofs} DoFs), reference RankOperator::apply, "
                       f"{BASIS.get(cfg_name, 'lagrange_gauss_lobatto')} basis, "
                       f"W={self.W}, R={self.n_ranks} threaded ranks (run_ranks + "
                       f"GhostExchanger), {self.inner} applies per step")

    def step(self):
        """DoF/s of one timed step (self.inner applies)."""
        return self.n_dofs * self.inner / self.world.time(self.inner)

    def rate(self, reps=11):
        """~10 s of CPU work: median of reps steps."""
        return statistics.median(self.step() for _ in range(reps))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dgx", choices=["dgx", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--cells", type=int, default=None, help="override cells per direction")
    ap.add_argument("--degree", type=int, default=None,
                    help="override the polynomial degree (C2 degree sweep p=1..10)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: n x n x (n * N) cells over N GPUs (z-slabs of n^3 each)")
    ap.add_argument("--ref-cells", type=int, default=None,
                    help="cells per direction of the reference CPU sample (default 16 in 3D)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_env()
    d, n, p, periodic, kind, coef, prec, seed, label = CONFIGS[args.config]
    p_config = p
    if args.degree:
        p = args.degree
    if args.config == "sweep":
        n = SWEEP_CELLS[p]
        p_config = None
        label = label.replace("n^3", f"{n}^3").replace("3D degree sweep", f"3D degree sweep p={p}")
    if args.cells:
        n = args.cells
    cells = [n] * d
    if args.weak:
        cells[-1] = n * ws
        label += f" (weak scaling: {n}^{d} cells per GPU)"
    n_dofs = int(np.prod(cells)) * (p + 1) ** d
    metric = ("DG advection apply throughput (DoFs/s)" if ADVECTION.get(args.config)
              else "DG Laplacian apply throughput (DoFs/s)")
    config = {"workload": label, "cells": cells, "degree": p, "n_dofs": n_dofs,
              "basis": BASIS.get(args.config, "lagrange_gauss_lobatto"),
              "geometry_variant": VARIANT.get(args.config, "g3"),
              "seed": seed, "partition": f"contiguous lexicographic slabs x{args.gpus}",
              "l2": "inputs larger than L2 (no flush)"}

    scaling = "weak" if args.weak else "strong"
    if args.impl == "reference":
        if rank != 0:
            return
        rb = RefBench(args.config, sample_cells=args.ref_cells, degree=p)
        for _ in range(args.warmup):
            rb.step()
        # one step = rb.inner applies of the sample; ms_per_step is the
        # measured wall time of such a step (median), value its DoF rate
        step_s = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            rb.world.time(rb.inner)
            step_s.append(time.perf_counter() - t0)
        t_step = statistics.median(step_s)
        val = rb.n_dofs * rb.inner / t_step
        info = {"cores": rb.n_ranks, "sample": rb.sample}
        out = {"metric": metric, "value": val, "unit": "DoF/s", "impl": "reference",
               "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": t_step * 1e3, "higher_is_better": True,
               "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": config,
               "measured": {"cells": rb.cells, "n_dofs": rb.n_dofs, "applies_per_step": rb.inner,
                            "note": "the reference CPU apply on a bounded sample of the workload "
                                    "(same configuration, measured cell count above); value is "
                                    "its DoF/s, ms_per_step the measured wall time of one step"},
               "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": info["cores"],
                                "kind": "reference", "sample": info["sample"]},
               "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_1711_03590_b200 as dgx

    torch.cuda.set_device(local)
    if ws > 1:
        # NCCL's INIT log (ranks, transports, NVLS) stays visible to the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t_setup = time.time()
    mesh = (dgx.make_box_mesh(d, cells, 0.05, periodic, 2) if kind == "mesh"
            else dgx.make_box_mesh(d, cells, 0.0, periodic, 1))
    faces = dgx.enumerate_faces(mesh)
    part = dgx.partition_cells(mesh, ws)
    dgx.assign_face_owners(mesh, faces, part)
    geo = (dgx.Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1" if coef else None)
           if kind == "vertex" else dgx.Geometry(source="mesh"))
    adv = ADVECTION.get(args.config)
    op = dgx.RankOperator(mesh, part, faces, geo, dgx.OperatorConfig(
        d=d, p=p, precision=prec, basis=BASIS.get(args.config, "lagrange_gauss_lobatto"),
        kind="advection" if adv else "laplacian", velocity=adv or (1.0, 1.0, 1.0),
        geometry=VARIANT.get(args.config, "g3")),
        rank, device=local)
    lay = op.layout()
    hooks = None
    if ws > 1:
        uid = [dgx.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        hooks = dgx.NcclExchanger(op, uid[0])
    del faces
    st = op.stats()
    dt = torch.float32 if prec == "fp32" else torch.float64
    esize = 4 if prec == "fp32" else 8
    nq = lay.dofs_per_cell
    # input: U[-1,1] from seed (std::mt19937 convention), this rank's slab
    # plus its ghost cells (gathered from the same global stream)
    b, e = lay.owned_cell_begin, lay.owned_cell_begin + lay.n_owned_cells
    x_owned = dgx.random_vector(e * nq, seed)[b * nq:]
    u_host = torch.empty(lay.total_size, dtype=dt).pin_memory()
    u_host[: lay.owned_size] = torch.from_numpy(x_owned).to(dt)
    del x_owned
    u = u_host.to(f"cuda:{local}")
    y = torch.empty_like(u)
    y_host = torch.empty(lay.total_size, dtype=dt).pin_memory()
    stream = torch.cuda.current_stream()
    t_setup = time.time() - t_setup

    def step():
        op.apply(u, y, hooks=hooks, stream=stream)

    def barrier():
        # drain this rank's exchange streams before the process group's own
        # collective starts: the exchanger's communicator and torch's never
        # have kernels in flight at the same time
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # working sets that fit in L2 (126 MB; small parity-size configurations
    # such as C1 / C2) are timed step by step with an L2 flush (a 512 MB write)
    # between steps, outside the events; larger ones back to back
    work_bytes = st["bytes_vectors"] + st["bytes_cell_geometry"] + st["bytes_face_geometry"]
    flush = None
    if work_bytes < 2 * L2_BYTES:
        flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")
        config["l2"] = (f"L2 flushed between timed steps (working set "
                        f"{work_bytes / 1e6:.0f} MB < 2x L2)")
    def load():  # ~0.3 s of the same applies, enqueued asynchronously
        n_load = max(1, int(300.0 / max(first_ms, 1e-3)))
        for _ in range(min(n_load, 2000)):
            step()

    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_a.record(stream)
    step()
    ev_b.record(stream)
    ev_b.synchronize()
    first_ms = ev_a.elapsed_time(ev_b)
    if ws > 1:
        # every rank must enqueue the same number of applies (each one posts
        # sends / receives to its neighbours): agree on the slowest rank's time
        fm = torch.tensor([first_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(fm, op=dist.ReduceOp.MAX)
        first_ms = float(fm.item())
    with ClockSampler(local, load=load if first_ms * args.steps < 1000.0 else None) as clk:
        barrier()
        if flush is None:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            barrier()
            t_ms = ev0.elapsed_time(ev1)
        else:
            evs = []
            with torch.cuda.stream(stream):
                for _ in range(args.steps):
                    flush.zero_()
                    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    step()
                    bb.record(stream)
                    evs.append((a, bb))
            barrier()
            t_ms = sum(a.elapsed_time(bb) for a, bb in evs)
    # per-step (= per-launch at N=1) durations for the roofline
    times = []
    for _ in range(min(args.steps, 5)):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.zero_()
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        bb.record(stream)
        bb.synchronize()
        times.append(a.elapsed_time(bb))
    t_max = torch.tensor([t_ms], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_ms = float(t_max.item())
    ms_per_step = t_ms / args.steps
    value = n_dofs / (ms_per_step * 1e-3)

    # end to end through the public API with host buffers: H2D of u, apply,
    # D2H of y every step
    e2e = None
    if not args.no_e2e:
        h2d = lay.total_size * esize if ws == 1 else lay.owned_size * esize
        d2h = lay.owned_size * esize
        if ws == 1 and prec == "fp64":
            # the public host-buffer call (dgx_apply_host: z-slab pipeline of
            # H2D / apply / D2H on three streams); blocking, so it is timed
            # by the host clock around synchronized calls
            op.apply_host(u_host, y_host)  # first call builds the pipeline state
            torch.cuda.synchronize()
            barrier()
            w0 = time.perf_counter()
            for _ in range(args.steps):
                op.apply_host(u_host, y_host)
            torch.cuda.synchronize()
            te = torch.tensor([(time.perf_counter() - w0) * 1e3], dtype=torch.float64,
                              device=f"cuda:{local}")
        else:
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                u[: h2d // esize].copy_(u_host[: h2d // esize], non_blocking=True)
                step()
                y_host[: d2h // esize].copy_(y[: d2h // esize], non_blocking=True)
            e1.record(stream)
            barrier()
            te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_dofs / (float(te.item()) / args.steps * 1e-3), "unit": "DoF/s",
               "h2d_bytes_per_step": int(h2d) * ws, "d2h_bytes_per_step": int(d2h) * ws}

    hbm, hbm_kind = peaks()
    alg_bytes = st["bytes_vectors"] + st["bytes_cell_geometry"] + st["bytes_face_geometry"]
    launch_ms = statistics.median(times)
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    # the binding resource: HBM bytes vs FP64 flops (reference counter flops,
    # SURVEY.md s.8d), whichever takes longer at its peak
    fpk, fpk_kind = fp64_peak(prec)
    ref_fpd = REF_FLOPS_PER_DOF.get(args.config, 0.0)
    if p != p_config:  # degree override: the reference counter values per degree
        ref_fpd = (C2_FLOPS_PER_DOF.get(p, 0.0) if args.config == "c2"
                   else SWEEP_FLOPS_PER_DOF.get(p, 0.0) if d == 3 else 0.0)
    flops = ref_fpd * lay.owned_size
    t_hbm = alg_bytes / (hbm * 1e9)
    t_fp64 = flops / (fpk * 1e12)
    if t_fp64 > t_hbm:
        achieved_f = flops / (launch_ms * 1e-3) / 1e12
        roofline = {"bound": prec, "achieved": achieved_f, "peak": fpk, "unit": "TFLOP/s",
                    "frac": achieved_f / fpk, "traffic": traffic, "peak_source": fpk_kind,
                    "algorithmic_flops_per_launch": flops,
                    "hbm_achieved_gbs": achieved, "hbm_frac": achieved / hbm}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic, "peak_source": hbm_kind,
                    "fp64_tflops": flops / (launch_ms * 1e-3) / 1e12}
    roofline.update({"algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_dof": alg_bytes / (lay.owned_size), "launch_ms": launch_ms,
                     "fp64_flops_per_dof_ref_counters": ref_fpd or None})

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            rb = RefBench(args.config, sample_cells=args.ref_cells, degree=p)
            cpu = {"value": rb.rate(), "unit": "DoF/s", "cores": rb.n_ranks,
                   "kind": "reference", "sample": rb.sample + ", median of 11 steps"}
        except Exception as ex:  # reported, never silently replaced
            cpu = {"value": None, "unit": "DoF/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if ws > 1:
        # tear the communicators down first: with NCCL_DEBUG=INFO their log
        # lines go to stdout, and the JSON line must be the last one
        dist.barrier()
        clk_summary = clk.summary()
        n_send_plans = len(op.plans("send"))
        del hooks
        import gc
        gc.collect()
        dist.destroy_process_group()
        if rank == 0:
            time.sleep(2.0)  # let the other ranks' teardown lines out first
    else:
        clk_summary = clk.summary()
        n_send_plans = 0
    if rank == 0:
        out = {"metric": metric, "value": value, "unit": "DoF/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
               "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
               "config": config, "e2e": e2e,
               "gpu_launches": int(args.steps * st["kernel_launches_per_apply"] +
                                   (args.steps * (1 + n_send_plans) if ws > 1 else 0)),
               "roofline": roofline, "cpu_baseline": cpu, "clocks": clk_summary,
               "setup_s": t_setup}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
