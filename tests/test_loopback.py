"""GPU: the native multi-rank data plane on one GPU.

R rank operators live in one process on cuda:0, each with the native device
exchanger (the same code bench.py --gpus N runs over NCCL: cell-list pack,
receives in place into u's ghost region or through the indexed unpack for
the Hermite-like two-layer plans, compress along the reversed routes,
accumulation in ascending neighbour rank, ghost region zeroed) over the
in-process loopback transport. Every rank runs dgx_apply with the
exchanger's hooks on its own host thread and its own stream -- the overlapped
schedule of Operator::apply (ghost-coupled cells on a high-priority stream,
compress posted while the inner cells run). This is the reference's own
distributed_apply pattern (tests/test_ghost_exchange.cpp:63-87: run_ranks
threads + GhostExchanger, ghost_exchange.cpp:300-398).

Checked: the gathered owned y against the reference's golden output (or the
C restatement oracle for R in {2, 3, 4, 8}), y's ghost region zero after
compress, u's ghost region equal to the neighbours' values, bitwise
repeatability across applies, fp32 at 1e-5.
"""
import threading

import numpy as np
import pytest

from conftest import Case, golden_names, rel_l2, rel_linf

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5
MULTI = [n for n in golden_names() if Case(n).n_ranks > 1]


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


def _dgx():
    import paper_1711_03590_b200 as m
    return m


def _geometry(c):
    G = _dgx().Geometry
    if c.vertex:
        return G(source="vertex_bump", vertex_bump_eps=c.eps,
                 coefficient="a1" if c.coefficient else None)
    return G(source="mesh")


def build_ranks(d, cells, p, n_ranks, amplitude=0.0, periodic=False, m=1, basis="lagrange_gauss_lobatto",
                geometry=None, kind="laplacian", velocity=(1.0, 1.0, 1.0), precision="fp64"):
    D = _dgx()
    mesh = D.make_box_mesh(d, cells, amplitude, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, n_ranks)
    D.assign_face_owners(mesh, faces, part)
    cfg = D.OperatorConfig(d=d, p=p, basis=basis, kind=kind, velocity=velocity, precision=precision)
    return [D.RankOperator(mesh, part, faces, geometry or D.Geometry(source="mesh"), cfg, r)
            for r in range(n_ranks)]


def loopback_apply(torch, ops, x, repeats=1, dtype=None, exs=None):
    """Every rank: u = owned slice + NaN ghosts, y = NaN; dgx_apply with the
    loopback exchanger's hooks on its own thread and stream. Returns the
    gathered owned y of each repeat and the per-rank (u, y) of the last."""
    D = _dgx()
    dtype = dtype or torch.float64
    if exs is None:
        world = D.LoopbackWorld(len(ops))
        exs = [D.LoopbackExchanger(op, world) for op in ops]
    nq = ops[0].layout().dofs_per_cell
    us, ys, streams = [], [], []
    for op in ops:
        lay = op.layout()
        b = lay.owned_cell_begin
        u = torch.full((lay.total_size,), float("nan"), dtype=dtype, device="cuda")
        u[: lay.owned_size] = torch.tensor(x[b * nq:(b + lay.n_owned_cells) * nq], dtype=dtype)
        us.append(u)
        ys.append(torch.full_like(u, float("nan")))
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    results = []
    for _ in range(repeats):
        errs = [None] * len(ops)

        def run(r):
            try:
                ops[r].apply(us[r], ys[r], hooks=exs[r], stream=streams[r])
                streams[r].synchronize()
            except Exception as e:  # re-raised on the main thread
                errs[r] = e

        th = [threading.Thread(target=run, args=(r,)) for r in range(len(ops))]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        for e in errs:
            if e is not None:
                raise e
        torch.cuda.synchronize()
        y = np.concatenate([ys[r][: op.layout().owned_size].double().cpu().numpy()
                            for r, op in enumerate(ops)])
        results.append(y)
    local = [(us[r].double().cpu().numpy(), ys[r].double().cpu().numpy()) for r in range(len(ops))]
    return results, local


def check_exchange_state(ops, local, x):
    nq = ops[0].layout().dofs_per_cell
    for op, (u, y) in zip(ops, local):
        lay = op.layout()
        # compress leaves y clean: ghost region zero
        assert np.all(y[lay.owned_size:] == 0.0)
        # the update delivered exactly the planned ghost dofs
        planned = np.zeros(lay.total_size, bool)
        for _, ix in op.plan_values("recv"):
            planned[ix] = True
        gx = np.concatenate([x[g * nq:(g + 1) * nq] for g in lay.ghost_global_cells]) \
            if len(lay.ghost_global_cells) else np.zeros(0)
        ug = u[lay.owned_size:]
        pg = planned[lay.owned_size:]
        assert np.array_equal(ug[pg], gx[pg])
        assert np.all(np.isnan(ug[~pg]))


@pytest.mark.parametrize("name", MULTI)
def test_loopback_golden(torch, name):
    """Every multi-rank golden fixture (1-7 ranks, GL / Gauss / Hermite-like
    two-layer plans, periodic wrap neighbours, ragged slabs, advection)
    through the native exchanger against the reference's output."""
    c = Case(name)
    D = _dgx()
    mesh = D.make_box_mesh(c.d, c.cells, c.amplitude, c.periodic, c.m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, c.n_ranks)
    D.assign_face_owners(mesh, faces, part)
    cfg = D.OperatorConfig(d=c.d, p=c.p, basis=c.basis_name, kind=c.kind, velocity=c.velocity,
                           variable_velocity=bool(c.velocity_field))
    ops = [D.RankOperator(mesh, part, faces, _geometry(c), cfg, r) for r in range(c.n_ranks)]
    if c.velocity_field:
        from test_gpu import set_field_velocity
        for op in ops:
            set_field_velocity(op, c.d)
    x = c.g[f"x{c.seeds[0]}"]
    ref = c.g[f"y{c.seeds[0]}"]
    (y1, y2), local = loopback_apply(torch, ops, x, repeats=2)
    assert rel_linf(y1, ref) < TOL64 and rel_l2(y1, ref) < TOL64
    assert np.array_equal(y1, y2), "exchanged apply not bitwise repeatable"
    check_exchange_state(ops, local, x)


@pytest.mark.parametrize("R", [2, 3, 4, 8])
@pytest.mark.parametrize("basis,p", [("lagrange_gauss_lobatto", 5), ("hermite_like", 4),
                                     ("lagrange_gauss", 3)])
def test_loopback_ranks(torch, R, basis, p):
    """R in {2, 3, 4, 8} on an 4 x 5 x 16 deformed Dirichlet mesh (slabs of
    10, 6.7, 5 and 2.5 z-layers: ragged partitions, interface cells split
    between face owners) against the C restatement oracle."""
    from oracle import oracle as O
    cells = [4, 5, 16]
    ops = build_ranks(3, cells, p, R, amplitude=0.05, m=2, basis=basis)
    b = {"lagrange_gauss_lobatto": 0, "lagrange_gauss": 1, "hermite_like": 2}[basis]
    P = O.Problem(3, cells, p, deform=("reference", 0.05, 2), basis=b)
    x = _dgx().random_vector(int(np.prod(cells)) * (p + 1) ** 3, 11)
    ref = P.apply(x)
    (y,), local = loopback_apply(torch, ops, x)
    assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64
    check_exchange_state(ops, local, x)


@pytest.mark.parametrize("R", [2, 4])
def test_loopback_periodic_vertex_coef(torch, R):
    """C4 shape: BASELINE vertex deformation with the folded a(x), periodic
    in z (rank 0 and rank R-1 exchange across the wrap)."""
    from oracle import oracle as O
    cells, p = [3, 4, 8], 5
    D = _dgx()
    geo = D.Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1")
    mesh = D.make_box_mesh(3, cells, 0.0, True, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, R)
    D.assign_face_owners(mesh, faces, part)
    ops = [D.RankOperator(mesh, part, faces, geo, D.OperatorConfig(d=3, p=p), r) for r in range(R)]
    x = D.random_vector(int(np.prod(cells)) * (p + 1) ** 3, 3)
    ref = O.Problem(3, cells, p, periodic=True, deform=("vertex", 0.1), coefficient=True).apply(x)
    (y,), local = loopback_apply(torch, ops, x)
    assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64
    check_exchange_state(ops, local, x)


@pytest.mark.parametrize("basis", ["lagrange_gauss_lobatto", "hermite_like"])
def test_loopback_fp32(torch, basis):
    """fp32 operators: messages of 4-byte values, the same plans."""
    from oracle import oracle as O
    cells, p, R = [4, 4, 8], 4, 3
    ops = build_ranks(3, cells, p, R, amplitude=0.05, m=2, basis=basis, precision="fp32")
    b = {"lagrange_gauss_lobatto": 0, "hermite_like": 2}[basis]
    x = _dgx().random_vector(int(np.prod(cells)) * (p + 1) ** 3, 5)
    ref = O.Problem(3, cells, p, deform=("reference", 0.05, 2), basis=b).apply(x)
    (y,), local = loopback_apply(torch, ops, x, dtype=torch.float32)
    assert rel_linf(y, ref) < TOL32 and rel_l2(y, ref) < TOL32
    for op, (u, yl) in zip(ops, local):
        assert np.all(yl[op.layout().owned_size:] == 0.0)


def test_loopback_errors(torch):
    """A bad apply fails before any hook runs (the exchanger is not left in
    flight: the next, correct apply works); plain hooks errors surface as the
    reference's exception classes."""
    D = _dgx()
    ops = build_ranks(3, [2, 2, 4], 3, 2)
    world = D.LoopbackWorld(2)
    exs = [D.LoopbackExchanger(op, world) for op in ops]
    lay = ops[0].layout()
    u = torch.zeros(lay.total_size, dtype=torch.float64, device="cuda")
    with pytest.raises(D.DgxInvalidArgument):
        ops[0].apply(u, u, hooks=exs[0])  # u == y: rejected before the update is posted
    f = torch.zeros(lay.total_size, dtype=torch.float32, device="cuda")
    with pytest.raises(D.DgxInvalidArgument):
        ops[0].apply(f, torch.zeros_like(f), hooks=exs[0])
    # the same exchangers: nothing was left in flight by the failed calls
    x = D.random_vector(16 * 64, 1)
    from oracle import oracle as O
    ref = O.Problem(3, [2, 2, 4], 3).apply(x)
    (y,), _ = loopback_apply(torch, ops, x, exs=exs)
    assert rel_linf(y, ref) < TOL64


def test_nccl_transport_single_rank(torch):
    """The NCCL transport with a one-rank communicator: libnccl resolves (the
    library torch loaded), ncclCommInitRank, grouped calls with no peers; an
    apply with the exchanger's hooks equals the plain apply. (More ranks need
    more GPUs: the multi-rank data plane runs over the loopback transport above.)"""
    D = _dgx()
    ops = build_ranks(3, [3, 3, 4], 5, 1, geometry=D.Geometry(source="vertex_bump", vertex_bump_eps=0.1))
    op = ops[0]
    ex = D.NcclExchanger(op, D.nccl_unique_id())
    x = D.random_vector(op.layout().total_size, 5)
    u = torch.tensor(x, device="cuda")
    y0, y1 = torch.empty_like(u), torch.empty_like(u)
    op.apply(u, y0)
    op.apply(u, y1, hooks=ex)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
