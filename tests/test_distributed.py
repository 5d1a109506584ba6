"""CPU, multi-process (gloo, world_size 2 and 3): the N>1 exchange protocol.

Each process builds its rank's layout and plans with the product host code
(libdgx.so, host-only operator), runs the ghost update and compress through
paper_1711_03590_b200.exchange.TorchExchanger over torch.distributed/gloo,
and uses the C restatement oracle as the compute stand-in for the device
kernel (test infrastructure). The gathered result must match the reference's
golden output (single-rank and its own threaded-rank runs).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import Case, rel_linf

CASES = ["def2d_periodic_p2_r4", "c3_vertex_p4_r3", "def3d_p3_m2_r2", "c4_vertex_coef_p5_r2",
         "cart3d_ragged_p4_r3", "herm3d_p5_m2_r3", "herm_c4_vertex_coef_p5_r2",
         "gauss3d_p3_m2_r2"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_03590_b200 as dgx
        from paper_1711_03590_b200.exchange import TorchExchanger, exchange_apply
        from oracle import oracle as O
        c = Case(name) if isinstance(name, str) else LiveCase(*name)
        mesh = dgx.make_box_mesh(c.d, c.cells, c.amplitude, c.periodic, c.m)
        faces = dgx.enumerate_faces(mesh)
        part = dgx.partition_cells(mesh, world)
        dgx.assign_face_owners(mesh, faces, part)
        op = dgx.RankOperator(mesh, part, faces, dgx.Geometry(),
                              dgx.OperatorConfig(d=c.d, p=c.p, basis=c.basis_name),
                              rank, device=-1)
        lay = op.layout()
        ex = TorchExchanger.from_operator(op)
        P = O.Problem(c.d, c.cells, c.p, periodic=c.periodic, deform=c.deform(),
                      coefficient=c.coefficient, n_ranks=world, basis=c.basis)
        nq = lay.dofs_per_cell
        x = c.g[f"x{c.seeds[0]}"]
        b, e = lay.owned_cell_begin, lay.owned_cell_begin + lay.n_owned_cells
        u = torch.zeros(lay.total_size, dtype=torch.float64)
        u[: lay.owned_size] = torch.from_numpy(x[b * nq:e * nq])
        u[lay.owned_size:] = float("nan")  # must be overwritten by the update
        y = torch.zeros_like(u)

        def phase1(uu, yy):
            pass

        def phase2(uu, yy):
            # oracle stand-in for the device kernel: rank-local apply with the
            # ghost values delivered by the update
            got = torch.zeros(lay.total_size, dtype=torch.bool)
            for _, ix in op.plan_values("recv"):
                got[torch.from_numpy(ix)] = True
            assert not torch.isnan(uu[got]).any(), "ghost update incomplete"
            # only the planned dofs travel (whole cells, or two layers per
            # coupled face for the Hermite-like basis); the rest stays unset
            # and must not be read
            ghost_nan = torch.isnan(uu[lay.owned_size:])
            if c.basis == 2:
                assert bool(ghost_nan[~got[lay.owned_size:]].all())
            else:
                assert not bool(ghost_nan.any())
            v = torch.where(got | (torch.arange(lay.total_size) < lay.owned_size), uu,
                            torch.zeros_like(uu))
            yy.copy_(torch.from_numpy(P.apply_rank_local(rank, v.numpy())))

        exchange_apply(ex, phase1, phase2, u, y)
        assert torch.all(y[lay.owned_size:] == 0)
        out = [None] * world
        dist.all_gather_object(out, (b, y[: lay.owned_size].numpy()))
        if rank == 0:
            full = np.zeros_like(x)
            for bb, part_y in out:
                full[bb * nq: bb * nq + part_y.size] = part_y
            q.put(rel_linf(full, c.g[f"y{c.seeds[0]}"]))
    except Exception as ex_:  # surface worker failures to the test
        q.put(repr(ex_))
        raise
    finally:
        dist.destroy_process_group()


class LiveCase:
    """A Cartesian configuration without a fixture: x seeded, y from the
    single-rank oracle (pinned against the reference in test_oracle.py)."""

    def __init__(self, d, cells, p, periodic, basis):
        from oracle import oracle as O
        self.d, self.cells, self.p, self.periodic = d, list(cells), p, periodic
        self.amplitude, self.m, self.coefficient = 0.0, 1, False
        self.basis = basis
        self.basis_name = ("lagrange_gauss_lobatto", "lagrange_gauss", "hermite_like")[basis]
        self.seeds = [1]
        P = O.Problem(d, self.cells, p, periodic=periodic, deform=None, n_ranks=1, basis=basis)
        x = O.random_vector(P.n_dofs, 4242 + p)
        self.g = {"x1": x, "y1": P.apply(x)}

    def deform(self):
        return None


# one cell per rank on a periodic line of cells: a rank's two neighbours in z
# are the same ghost cell (world 2), or the ghosts of both sides differ (world 3)
DEGENERATE = [(3, (1, 1, 3), 3, True, 0), (3, (1, 1, 3), 4, True, 2), (2, (1, 3), 5, True, 0)]


@pytest.mark.parametrize("cfg", DEGENERATE, ids=lambda c: f"d{c[0]}p{c[2]}b{c[4]}")
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_degenerate(cfg, world):
    test_gloo_exchange_matches_reference(cfg, world)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_matches_reference(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), res
    assert isinstance(res, float), res
    assert res < 1e-12
