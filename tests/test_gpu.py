"""GPU parity: the CUDA path (through the C ABI) against the reference.

* golden fixtures produced by the unmodified reference (single rank and
  R ranks; per-rank results through the split phases + a serial compress,
  the reference's SerialRanks pattern, tests/test_operators.cpp:446-535);
* the C restatement oracle on random configurations, p = 1..10, 2D and 3D,
  Cartesian / curved / BASELINE vertex deformation / folded a(x);
* device geometry against the reference's precompute_geometry;
* size-independent properties at BASELINE sizes (symmetry, linearity,
  constants in the kernel on periodic meshes, bitwise determinism);
* fp32 against fp64 at 1e-5.
Tolerances: rel L_inf and rel L2 <= 1e-12 (fp64), 1e-5 (fp32), as north_star
states.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import Case, cuda_available, golden_names, rel_l2, rel_linf

pytestmark = pytest.mark.gpu

NAMES = golden_names()
TOL64 = 1e-12
TOL32 = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


@pytest.fixture
def free_hbm(torch):
    """Full-size tests: release the operators and cached blocks of earlier
    tests first (the library allocates with cudaMalloc, outside torch's cache)."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    torch.cuda.empty_cache()


def dgx():
    import paper_1711_03590_b200 as m
    return m


def geometry_of(c: Case):
    G = dgx().Geometry
    if c.vertex:
        return G(source="vertex_bump", vertex_bump_eps=c.eps,
                 coefficient="a1" if c.coefficient else None)
    return G(source="mesh")


def build(c: Case, rank=0, n_ranks=None, precision="fp64", p=None):
    D = dgx()
    mesh = D.make_box_mesh(c.d, c.cells, c.amplitude, c.periodic, c.m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, n_ranks or c.n_ranks)
    D.assign_face_owners(mesh, faces, part)
    cfg = D.OperatorConfig(d=c.d, p=p or c.p, precision=precision, basis=c.basis_name,
                           kind=c.kind, velocity=c.velocity,
                           variable_velocity=bool(c.velocity_field))
    op = D.RankOperator(mesh, part, faces, geometry_of(c), cfg, rank)
    if c.velocity_field:
        set_field_velocity(op, c.d)
    return op, part


def set_field_velocity(op, d):
    """The harness's variable transport field at the device quadrature points."""
    import torch as t
    from oracle import reflib as R
    cc = t.tensor(R.test_velocity(d, op.quadrature_points("cells")).ravel(), device="cuda")
    cf = t.tensor(R.test_velocity(d, op.quadrature_points("faces")).ravel(), device="cuda")
    op.set_velocity(cc, cf)
    t.cuda.synchronize()


def apply_single(torch, op, x, dtype=None):
    dtype = dtype or torch.float64
    u = torch.tensor(x, dtype=dtype, device="cuda")
    y = torch.empty_like(u)
    op.apply(u, y)
    torch.cuda.synchronize()
    return y.double().cpu().numpy()


def apply_serial_ranks(torch, ops, parts, x, nq, return_local=False, planned_only=False):
    """SerialRanks (reference tests/test_operators.cpp:446-535): ghost fill by
    copy, both phases on the device per rank, compress on the host.
    planned_only: only the dofs of the receive plans are filled (what the
    exchange ships), every other ghost value is NaN and must not be read."""
    y = np.zeros_like(x)
    local = []
    for r, op in enumerate(ops):
        lay = op.layout()
        b = lay.owned_cell_begin
        e = b + lay.n_owned_cells
        u_loc = np.concatenate([x[b * nq:e * nq]] +
                               [x[g * nq:(g + 1) * nq] for g in lay.ghost_global_cells])
        if planned_only:
            keep = np.zeros(u_loc.size, bool)
            keep[: lay.owned_size] = True
            for _, ix in op.plan_values("recv"):
                keep[ix] = True
            u_loc = np.where(keep, u_loc, np.nan)
        u = torch.tensor(u_loc, device="cuda")
        yl = torch.full_like(u, float("nan"))
        op.apply_phase(1, u, yl)
        op.apply_phase(2, u, yl)
        torch.cuda.synchronize()
        y_loc = yl.cpu().numpy()
        local.append((u_loc, y_loc))
        y[b * nq:e * nq] += y_loc[: (e - b) * nq]
        for i, g in enumerate(lay.ghost_global_cells):
            y[g * nq:(g + 1) * nq] += y_loc[(e - b + i) * nq:(e - b + i + 1) * nq]
    return (y, local) if return_local else y


@pytest.mark.parametrize("name", NAMES)
def test_golden_single_rank(torch, name):
    c = Case(name)
    op, _ = build(c, n_ranks=1)
    for s in c.seeds:
        y = apply_single(torch, op, c.g[f"x{s}"])
        ref = c.g[f"y{s}"]
        assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64, (rel_linf(y, ref), rel_l2(y, ref))


@pytest.mark.parametrize("name", [n for n in NAMES if n.endswith(("_r2", "_r3", "_r4", "_r7"))])
def test_golden_rank_partitioned(torch, name):
    from oracle import oracle as O
    c = Case(name)
    ops, parts = [], []
    for r in range(c.n_ranks):
        op, part = build(c, rank=r)
        ops.append(op)
        parts.append(part)
    nq = (c.p + 1) ** c.d
    x = c.g[f"x{c.seeds[0]}"]
    y, local = apply_serial_ranks(torch, ops, parts, x, nq, return_local=True,
                                  planned_only=c.basis == 2 or c.kind == "advection")
    assert rel_linf(y, c.g[f"y{c.seeds[0]}"]) < TOL64
    if c.kind == "advection":
        from oracle import reflib as R
        if not R.available():
            return
        w = R.World(c.d, c.cells, c.p, n_ranks=c.n_ranks, amplitude=c.amplitude,
                    mapping_degree=c.m, periodic=c.periodic,
                    basis={0: "gl", 1: "gauss", 2: "hermite"}[c.basis], kind="advection",
                    velocity=c.velocity, velocity_field=c.velocity_field)
        for r, (u_loc, y_loc) in enumerate(local):
            assert np.all(np.isfinite(y_loc))
            ref = w.apply_rank_local(r, np.nan_to_num(u_loc, nan=0.0))
            assert rel_linf(y_loc, ref) < TOL64
        return
    # per-rank state before compress (ghost slots hold remote contributions)
    P = O.Problem(c.d, c.cells, c.p, periodic=c.periodic, deform=c.deform(),
                  coefficient=c.coefficient, n_ranks=c.n_ranks, basis=c.basis)
    for r, (u_loc, y_loc) in enumerate(local):
        assert np.all(np.isfinite(y_loc))
        assert rel_linf(y_loc, P.apply_rank_local(r, np.nan_to_num(u_loc, nan=0.0))) < TOL64


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith(("c1", "def3d", "c3", "c4", "c5", "def2d_p3"))])
def test_device_geometry(torch, name):
    c = Case(name)
    if "geo_jxw" not in c.g:
        pytest.skip("no geometry in fixture")
    op, _ = build(c, n_ranks=1)
    d, k = c.d, c.p + 1
    nq, nqf = k ** d, k ** (d - 1)
    cg = op.device_geometry(0)
    nrec = 1 if bool(c.g.get("compressed", False)) else nq
    nc = int(np.prod(c.cells))
    cg = cg.reshape(nc, d * d + 1, nrec)
    jit = c.g["geo_inv_jac_t"].reshape(nc, nrec, d * d).transpose(0, 2, 1)
    jxw = c.g["geo_jxw"].reshape(nc, nrec)
    tol = 1e-14 if c.coefficient else 0.0
    assert rel_linf(cg[:, : d * d, :], jit) <= tol
    assert rel_linf(cg[:, d * d, :], jxw) <= tol
    fids = op.device_geometry(3).astype(np.int64)
    if nrec == 1:
        # Cartesian: compressed face records, JxW_f = record * prod_t w[q_t]
        from oracle import oracle as O
        _, w = O.gauss(k)
        wqf = np.ones(nqf)
        for q in range(nqf):
            idx = q
            for _a in range(d - 1):
                wqf[q] *= w[idx % k]
                idx //= k
        fr = op.device_geometry(1).reshape(-1, 2 * d + 1, 1)
        fg = np.concatenate([fr[:, :1, :] * wqf[None, None, :],
                             np.repeat(fr[:, 1:, :], nqf, axis=2)], axis=1)
        tol = 1e-15
    else:
        fg = op.device_geometry(1).reshape(-1, 2 * d + 1, nqf)
    assert rel_linf(fg[:, 0, :], c.g["geo_face_jxw"].reshape(-1, nqf)[fids]) <= tol
    jni = c.g["geo_face_jni"].reshape(-1, nqf, d)[fids].transpose(0, 2, 1)
    jne = c.g["geo_face_jne"].reshape(-1, nqf, d)[fids].transpose(0, 2, 1)
    assert rel_linf(fg[:, 1:1 + d, :], jni) <= tol
    assert rel_linf(fg[:, 1 + d:, :], jne) <= tol
    assert rel_linf(op.device_geometry(2), c.g["geo_penalty"][fids]) <= max(tol, 1e-15)


RANDOM = [
    # d, cells, p, periodic, deform, coefficient, ranks
    (2, [5, 4], p, bool(p % 2), ("reference", 0.05, 2), False, 1) for p in range(1, 11)
] + [
    (3, [3, 3, 2], p, bool(p % 2), ("reference", 0.04, 2), False, 1) for p in range(1, 11)
] + [
    (3, [4, 3, 3], 4, False, ("vertex", 0.1), False, 3),
    (3, [3, 3, 4], 5, False, ("vertex", 0.1), True, 2),
    (3, [4, 4, 3], 6, True, None, False, 4),
    (2, [7, 5], 7, False, ("vertex", 0.1), True, 3),
    (3, [2, 2, 2], 10, False, ("vertex", 0.1), False, 1),
    (3, [1, 1, 3], 3, True, None, False, 1),
    # x-rows inside one CTA of the pencil-pair kernel (even k): faces between
    # consecutive tasks take the partner's trace from shared memory
    (3, [5, 2, 2], 5, True, ("reference", 0.04, 2), False, 1),
    (3, [2, 3, 3], 3, True, None, False, 1),
    (3, [6, 2, 2], 7, False, ("vertex", 0.1), True, 2),
    (3, [7, 2, 1], 9, True, ("reference", 0.04, 2), False, 1),
    # degenerate meshes: one periodic cell (each face pairs the cell with
    # itself; in the pair kernel the x partner is the cell itself), two cells
    # periodic in x (partner and periodic neighbour coincide), one-cell-thick
    # slabs, a single Dirichlet cell
    (3, [1, 1, 1], 5, True, None, False, 1),
    (3, [1, 1, 1], 4, True, None, False, 1),
    (3, [2, 1, 1], 3, True, None, False, 1),
    (3, [2, 1, 1], 5, True, ("vertex", 0.1), True, 1),
    (3, [1, 2, 1], 1, True, None, False, 1),
    (3, [1, 1, 1], 2, False, None, False, 1),
    (2, [1, 1], 4, True, None, False, 1),
    (2, [1, 9], 5, True, None, False, 1),
    (2, [9, 1], 3, True, ("vertex", 0.1), False, 1),
    # one cell per rank, periodic: a rank's two z neighbours are one ghost cell
    (3, [1, 1, 2], 3, True, None, False, 2),
    (3, [1, 1, 3], 5, True, None, False, 3),
    (2, [2, 1], 5, True, None, False, 2),
]


def _cfg_id(c):
    return (f"d{c[0]}p{c[2]}r{c[6]}{'P' if c[3] else 'D'}{c[4][0][0] if c[4] else 'C'}"
            f"{'a' if c[5] else ''}{'' if len(c) < 8 else '-' + c[7]}")


@pytest.mark.parametrize("cfg", RANDOM, ids=_cfg_id)
def test_random_configs_against_oracle(torch, cfg):
    run_random_config(torch, cfg)


# the reference default basis for the Laplacian at p >= 3 (Hermite-like,
# operators.cpp:27-41) and the Lagrange-Gauss collocation basis; multi-rank
# cases fill only the planned ghost dofs (two layers per coupled face)
RANDOM_BASES = [
    (3, [3, 3, 2], p, bool(p % 2), ("reference", 0.04, 2), False, 1, "hermite_like")
    for p in range(3, 11)
] + [
    (2, [5, 4], p, bool(p % 2), ("reference", 0.05, 2), False, 1, "hermite_like")
    for p in range(3, 11)
] + [
    (3, [4, 3, 3], 5, False, ("vertex", 0.1), True, 3, "hermite_like"),
    (3, [3, 4, 3], 4, True, None, False, 4, "hermite_like"),
    (2, [7, 5], 6, False, ("vertex", 0.1), False, 3, "hermite_like"),
    (3, [3, 3, 3], 8, False, ("reference", 0.05, 2), False, 2, "hermite_like"),
    (3, [5, 3, 2], 5, True, ("reference", 0.04, 2), False, 1, "hermite_like"),
    (3, [3, 3, 2], 2, False, ("reference", 0.04, 2), False, 2, "lagrange_gauss"),
    (3, [3, 2, 2], 5, True, None, False, 1, "lagrange_gauss"),
    (2, [5, 4], 7, False, ("vertex", 0.1), True, 3, "lagrange_gauss"),
    # degenerate meshes (one periodic cell; one cell per rank)
    (3, [1, 1, 1], 4, True, None, False, 1, "hermite_like"),
    (3, [1, 1, 2], 4, True, None, False, 2, "hermite_like"),
    (3, [1, 1, 1], 3, True, None, False, 1, "lagrange_gauss"),
]


@pytest.mark.parametrize("cfg", RANDOM_BASES, ids=_cfg_id)
def test_other_bases_against_oracle(torch, cfg):
    run_random_config(torch, cfg)


def run_random_config(torch, cfg):
    from oracle import oracle as O
    D = dgx()
    d, cells, p, periodic, deform, coef, nr = cfg[:7]
    basis = cfg[7] if len(cfg) > 7 else "lagrange_gauss_lobatto"
    P = O.Problem(d, cells, p, periodic=periodic, deform=deform, coefficient=coef, n_ranks=nr,
                  basis=O.BASIS[basis])
    amp = deform[1] if deform and deform[0] == "reference" else 0.0
    m = deform[2] if deform and deform[0] == "reference" else 1
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    geo = (D.Geometry(source="vertex_bump", vertex_bump_eps=deform[1], coefficient="a1" if coef else None)
           if deform and deform[0] == "vertex" else D.Geometry(source="mesh"))
    x = O.random_vector(P.n_dofs, 1000 + p)
    y_ref = P.apply(x)
    ops = []
    for r in range(nr):
        part = D.partition_cells(mesh, nr)
        D.assign_face_owners(mesh, faces, part)
        ops.append(D.RankOperator(mesh, part, faces, geo, D.OperatorConfig(d=d, p=p, basis=basis),
                                  r))
    if nr == 1:
        y = apply_single(torch, ops[0], x)
    else:
        y = apply_serial_ranks(torch, ops, None, x, (p + 1) ** d,
                               planned_only=basis == "hermite_like")
    assert rel_linf(y, y_ref) < TOL64 and rel_l2(y, y_ref) < TOL64, (rel_linf(y, y_ref), rel_l2(y, y_ref))


class SerialHooks:
    """dgx_hooks backed by ctypes callbacks; records the call order."""

    def __init__(self):
        from paper_1711_03590_b200 import _lib
        self.calls = []

        def mk(name):
            def fn(ctx, vec, stream):
                self.calls.append(name)
                return 0
            return _lib.HOOK_FN(fn)
        self._fns = [mk("start"), mk("finish"), mk("compress")]
        self._c = _lib.CHooks(None, *self._fns)

    def c_hooks(self):
        return self._c


def test_hooks_protocol(torch):
    c = Case("def3d_p3_m2_r2")
    op, _ = build(c, rank=0)
    n = op.layout().total_size
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(u)
    D = dgx()
    with pytest.raises(D.DgxLogicError):
        op.apply(u, y)  # ghosted layout without hooks (operators.cpp:238-240)
    h = SerialHooks()
    op.apply(u, y, hooks=h)
    torch.cuda.synchronize()
    assert h.calls == ["start", "finish", "compress"]
    with pytest.raises(D.DgxInvalidArgument):
        op.apply(u, u, hooks=h)


def test_apply_host_pointers(torch):
    c = Case("c5_cart_p6")
    op, _ = build(c, n_ranks=1)
    y = op.apply_host(c.g["x4"])
    assert rel_linf(y, c.g["y4"]) < TOL64


@pytest.mark.parametrize("periodic", [False, True])
def test_apply_host_pipeline_advection(torch, periodic):
    """The z-slab host pipeline runs the advection operator too (its
    neighbour reads cross z like the Laplacian's): same result as the
    device apply."""
    D = dgx()
    cells, p = [3, 2, 10], 4
    mesh = D.make_box_mesh(3, cells, 0.05, periodic, 2)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                        D.OperatorConfig(d=3, p=p, kind="advection", velocity=(0.3, -0.7, 1.1)), 0)
    x = D.random_vector(op.layout().total_size, 11)
    u = torch.tensor(x, device="cuda:0")
    yd = torch.empty_like(u)
    op.apply(u, yd)
    torch.cuda.synchronize()
    yh = op.apply_host(x)
    assert rel_linf(yh, yd.cpu().numpy()) < 1e-14


@pytest.mark.parametrize("periodic,p,cells", [(False, 3, [3, 2, 9]), (True, 5, [2, 3, 8]),
                                              (True, 4, [2, 2, 33])])
def test_apply_host_pipeline(torch, periodic, p, cells):
    """dgx_apply_host on single-rank 3D layouts pipelines H2D / apply / D2H
    over z-slabs (own task order per slab): same result as the device apply
    and the oracle, repeated calls and pinned torch buffers included."""
    from oracle import oracle as O
    D = dgx()
    mesh = D.make_box_mesh(3, cells, 0.0, periodic, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="vertex_bump", vertex_bump_eps=0.1),
                        D.OperatorConfig(d=3, p=p), 0)
    x = D.random_vector(op.layout().total_size, 7)
    ref = O.Problem(3, cells, p, periodic=periodic, deform=("vertex", 0.1)).apply(x)
    y1 = op.apply_host(x)
    assert rel_linf(y1, ref) < TOL64 and rel_l2(y1, ref) < TOL64
    u = torch.tensor(x, device="cuda:0")
    yd = torch.empty_like(u)
    op.apply(u, yd)
    torch.cuda.synchronize()
    assert rel_linf(y1, yd.cpu().numpy()) < 1e-14
    uh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(uh).pin_memory()
    for _ in range(2):
        yh.zero_()
        op.apply_host(uh, yh)
        assert np.array_equal(yh.numpy(), y1)


@pytest.mark.parametrize("name", ["c5_cart_p6", "c3_vertex_p4", "c1_periodic_cart_p3", "c2_dirichlet_cart_p10",
                                  "herm3d_p3_m2", "herm_c4_vertex_coef_p5_r2", "gauss2d_p2_periodic"])
def test_fp32_against_fp64_reference(torch, name):
    c = Case(name)
    op, _ = build(c, n_ranks=1, precision="fp32")
    s = c.seeds[0]
    y = apply_single(torch, op, c.g[f"x{s}"], dtype=torch.float32)
    assert rel_l2(y, c.g[f"y{s}"]) < TOL32


FP32_RANDOM = [
    # d, cells, p, periodic, deform, coefficient, basis (single rank)
    (3, [3, 3, 2], 5, False, ("vertex", 0.1), True, "lagrange_gauss_lobatto"),
    (3, [2, 2, 2], 4, True, ("reference", 0.04, 2), False, "lagrange_gauss_lobatto"),
    (2, [5, 4], 7, False, ("vertex", 0.1), False, "lagrange_gauss_lobatto"),
    (3, [3, 2, 2], 6, True, None, False, "hermite_like"),
    # degenerate meshes
    (3, [1, 1, 1], 5, True, None, False, "lagrange_gauss_lobatto"),
    (3, [2, 1, 1], 4, True, None, False, "lagrange_gauss_lobatto"),
    (2, [1, 1], 3, True, None, False, "lagrange_gauss_lobatto"),
]


@pytest.mark.parametrize("cfg", FP32_RANDOM, ids=lambda c: f"d{c[0]}p{c[2]}{c[6][:4]}")
def test_fp32_random_against_oracle(torch, cfg):
    """The fp32 apply (dgx_apply_f32) against the fp64 oracle, TOL32 in rel L2."""
    from oracle import oracle as O
    D = dgx()
    d, cells, p, periodic, deform, coef, basis = cfg
    P = O.Problem(d, cells, p, periodic=periodic, deform=deform, coefficient=coef, n_ranks=1,
                  basis=O.BASIS[basis])
    amp = deform[1] if deform and deform[0] == "reference" else 0.0
    m = deform[2] if deform and deform[0] == "reference" else 1
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    geo = (D.Geometry(source="vertex_bump", vertex_bump_eps=deform[1], coefficient="a1" if coef else None)
           if deform and deform[0] == "vertex" else D.Geometry(source="mesh"))
    op = D.RankOperator(mesh, part, faces, geo,
                        D.OperatorConfig(d=d, p=p, precision="fp32", basis=basis), 0)
    x = O.random_vector(P.n_dofs, 3000 + p)
    y = apply_single(torch, op, x, dtype=torch.float32)
    assert rel_l2(y, P.apply(x)) < TOL32


# Cartesian meshes, nodal bases: the tensor-product kernel (sipg_cart.cuh) against the
# oracle -- every degree in 2D and 3D, Dirichlet and periodic, 1-3 ranks (ghost-side
# tasks), all three bases, anisotropic cells (cells per direction differ on the unit box)
CART_TENSOR = (
    [(2, [5, 4], p, p % 2 == 0, None, False, 1 + p % 2) for p in range(1, 11)] +
    [(3, [3, 2, 4], p, p % 2 == 1, None, False, 1) for p in range(1, 8)] +
    [(3, [2, 2, 3], p, False, None, False, 3) for p in (2, 3, 6)] +
    [(3, [2, 2, 2], p, True, None, False, 2) for p in (8, 9, 10)] +
    [(3, [3, 2, 2], 4, False, None, False, 2, "lagrange_gauss"),
     (3, [2, 3, 2], 5, True, None, False, 1, "lagrange_gauss"),
     (2, [4, 3], 6, False, None, False, 2, "lagrange_gauss"),
     (2, [3, 3], 3, True, None, False, 1, "lagrange_gauss")] +
    # Hermite-like: two neighbour layers, sign-flipped tables, masked ghost cells
    [(3, [3, 2, 3], p, p % 2 == 0, None, False, 1 + p % 3, "hermite_like") for p in (3, 4, 5, 7, 10)] +
    [(2, [4, 5], p, p % 2 == 1, None, False, 1 + p % 2, "hermite_like") for p in (3, 6, 9)]
)


@pytest.mark.parametrize("cfg", CART_TENSOR, ids=lambda c: _cfg_id(c))
def test_cart_tensor_kernel(torch, cfg):
    D = dgx()
    d, cells, p = cfg[:3]
    basis = cfg[7] if len(cfg) > 7 else "lagrange_gauss_lobatto"
    mesh = D.make_box_mesh(d, cells, 0.0, cfg[3], 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                        D.OperatorConfig(d=d, p=p, basis=basis), 0)
    assert op.stats()["cartesian"] == 2  # the tensor-product kernel runs
    run_random_config(torch, cfg)


@pytest.mark.parametrize("cfg", [(2, [6, 5], 4, False), (2, [4, 4], 9, True), (3, [3, 3, 2], 3, True),
                                 (3, [2, 3, 3], 6, False), (3, [2, 2, 2], 10, False)],
                         ids=lambda c: f"d{c[0]}p{c[2]}")
def test_cart_tensor_kernel_fp32(torch, cfg):
    from oracle import oracle as O
    D = dgx()
    d, cells, p, periodic = cfg
    P = O.Problem(d, cells, p, periodic=periodic, deform=None, coefficient=False, n_ranks=1,
                  basis=O.BASIS["lagrange_gauss_lobatto"])
    mesh = D.make_box_mesh(d, cells, 0.0, periodic, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                        D.OperatorConfig(d=d, p=p, precision="fp32"), 0)
    assert op.stats()["cartesian"] == 2
    x = O.random_vector(P.n_dofs, 4000 + p)
    y = apply_single(torch, op, x, dtype=torch.float32)
    assert rel_l2(y, P.apply(x)) < TOL32


def test_cart_tensor_matches_collocation_kernel(torch, monkeypatch):
    """Same operator, two kernels: tensor-product vs the collocation CART kernel
    (DGX_NO_TENSOR) on a 3D Dirichlet mesh with anisotropic cells."""
    from oracle import oracle as O
    D = dgx()
    d, cells, p = 3, [5, 3, 4], 4
    mesh = D.make_box_mesh(d, cells, 0.0, False, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    x = O.random_vector(int(np.prod(cells)) * (p + 1) ** d, 77)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), D.OperatorConfig(d=d, p=p), 0)
    y_t = apply_single(torch, op, x)
    monkeypatch.setenv("DGX_NO_TENSOR", "1")
    op2 = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), D.OperatorConfig(d=d, p=p), 0)
    assert op2.stats()["cartesian"] == 1
    y_c = apply_single(torch, op2, x)
    assert rel_linf(y_t, y_c) < TOL64 and rel_l2(y_t, y_c) < TOL64


def big_problem(torch, d, n, p, periodic, geometry):
    D = dgx()
    mesh = D.make_box_mesh(d, n, 0.0, periodic, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    return D.RankOperator(mesh, part, faces, geometry, D.OperatorConfig(d=d, p=p))


def dot(a, b):
    return float((a * b).sum().item())


@pytest.mark.parametrize("shape", [
    ("C1", 3, 16, 3, True, "cart"),
    ("C3", 3, 64, 4, False, "vertex"),
    ("C2", 2, 256, 7, False, "cart"),
    # BASELINE sizes of the bench configurations (pencil-pair kernel; C5 odd k)
    ("C4", 3, 128, 5, False, "vertex_a"),
    ("C5", 3, 160, 6, False, "cart"),
])
def test_full_size_properties(torch, shape, free_hbm):
    """Properties that hold at any size: symmetry v.Au = u.Av, linearity,
    bitwise repeatability, and A 1 = 0 on periodic meshes (constants are in
    the kernel of the SIP Laplacian; GL nodal coefficients of 1 are 1)."""
    name, d, n, p, periodic, kind = shape
    D = dgx()
    geo = (D.Geometry(source="vertex_bump", vertex_bump_eps=0.1,
                      coefficient="a1" if kind == "vertex_a" else None)
           if kind.startswith("vertex") else D.Geometry())
    op = big_problem(torch, d, n, p, periodic, geo)
    N = op.layout().total_size
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    v = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Au, Av = torch.empty_like(u), torch.empty_like(u)
    op.apply(u, Au)
    op.apply(v, Av)
    scale = float(torch.linalg.norm(u) * torch.linalg.norm(Av))
    assert abs(dot(v, Au) - dot(u, Av)) < 1e-12 * scale
    assert dot(u, Au) > 0  # positive (semi-)definite
    w, Aw = 0.3 * u - 1.7 * v, torch.empty_like(u)
    op.apply(w, Aw)
    assert float(torch.linalg.norm(Aw - (0.3 * Au - 1.7 * Av))) < 1e-12 * float(torch.linalg.norm(Aw))
    Au2 = torch.empty_like(u)
    op.apply(u, Au2)
    assert torch.equal(Au, Au2)
    if periodic:
        one = torch.ones_like(u)
        A1 = torch.empty_like(u)
        op.apply(one, A1)
        assert float(A1.abs().max()) < 1e-11 * float(Au.abs().max())


def test_reference_adapter(torch):
    """tests/cpp/adapter_test: the reference's own fixtures (SingleRankOp,
    distributed_apply with GhostExchanger) with dgx_ref::RankOperator swapped
    in, against dg::RankOperator (rel L_inf <= 1e-12)."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "adapter_test")
    if not os.path.exists(exe):
        pytest.skip("adapter test not built (needs the reference headers)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout


@pytest.mark.parametrize("cfg", [(2, [4, 4], 3, 0.05, 2), (3, [3, 3, 3], 4, 0.05, 2), (3, [4, 4, 4], 2, 0.0, 1)])
def test_conjugate_gradient_against_reference(torch, cfg):
    """Device CG (dgx_conjugate_gradient) vs the reference
    conjugate_gradient(make_apply(op)) (solvers.cpp:24-68,189-206) on the
    same Dirichlet system: both converge to 1e-10, iteration counts agree to
    round-off, solutions agree to 1e-8."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    d, cells, p, amp, m = cfg
    D = dgx()
    w = R.World(d, cells, p, amplitude=amp, mapping_degree=m)
    b = R.random_vector(w.n_dofs, 17)
    x_ref, rep_ref = w.cg(b, 1e-10, 2000)
    mesh = D.make_box_mesh(d, cells, amp, False, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), D.OperatorConfig(d=d, p=p))
    bd = torch.tensor(b, device="cuda")
    xd = torch.empty_like(bd)
    rep = op.conjugate_gradient(bd, xd, rel_tol=1e-10, max_iterations=2000)
    assert rep["converged"] and rep_ref["converged"]
    assert rep["relative_residual"] <= 1e-10
    assert abs(rep["iterations"] - rep_ref["iterations"]) <= 2, (rep, rep_ref)
    assert rel_l2(xd.cpu().numpy(), x_ref) < 1e-8


def test_conjugate_gradient_contract(torch):
    D = dgx()
    c = Case("def3d_p3_m2_r2")
    op, _ = build(c, rank=0)
    n = op.layout().owned_size
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    with pytest.raises(D.DgxInvalidArgument):  # make_apply: single rank only
        op.conjugate_gradient(b, torch.empty_like(b))


RHS_CASES = [
    # d, cells, p, amplitude, m, periodic, ranks, basis
    (3, [3, 3, 3], 3, 0.05, 2, False, 1, "lagrange_gauss_lobatto"),
    (2, [4, 5], 4, 0.06, 3, False, 2, "hermite_like"),
    (3, [4, 4, 3], 5, 0.0, 1, False, 1, "hermite_like"),
    (3, [3, 3, 4], 2, 0.05, 2, False, 3, "lagrange_gauss"),
    (3, [2, 3, 4], 6, 0.04, 2, False, 2, "lagrange_gauss_lobatto"),
]
_RB = {"lagrange_gauss_lobatto": "gl", "lagrange_gauss": "gauss", "hermite_like": "hermite"}


@pytest.mark.parametrize("cfg", RHS_CASES, ids=lambda c: f"d{c[0]}p{c[2]}r{c[6]}-{c[7]}")
def test_assemble_rhs_against_reference(torch, cfg):
    """assemble_rhs (forcing + Dirichlet data, operators.cpp:266-282) with the
    manufactured data of the convergence study, per rank, against the
    reference; f and g evaluated at the device's quadrature points."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p, amp, m, periodic, nr, basis = cfg
    w = R.World(d, cells, p, n_ranks=nr, amplitude=amp, mapping_degree=m, periodic=periodic,
                basis=_RB[basis], manufactured=True)
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, nr)
    D.assign_face_owners(mesh, faces, part)
    for r in range(nr):
        op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                            D.OperatorConfig(d=d, p=p, basis=basis), r)
        xq = op.quadrature_points("cells")
        xf = op.quadrature_points("faces")
        f = torch.tensor(R.manufactured_forcing(d, xq).ravel(), device="cuda")
        g = torch.tensor(R.manufactured_solution(d, xf).ravel(), device="cuda")
        rhs = torch.full((op.layout().total_size,), float("nan"), dtype=torch.float64,
                         device="cuda")
        op.assemble_rhs(rhs, f, g)
        torch.cuda.synchronize()
        ref = w.rhs(r)
        got = rhs.cpu().numpy()
        assert rel_linf(got, ref) < TOL64 and rel_l2(got, ref) < TOL64, (rel_linf(got, ref),)


def test_quadrature_points_match_reference_geometry(torch):
    """Face quadrature points equal the reference GeometryCache::face_qpoints
    (geometry.cpp:415-453) bit for bit on a curved mesh."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p = 3, [3, 2, 3], 4
    w = R.World(d, cells, p, amplitude=0.05, mapping_degree=2)
    mesh = D.make_box_mesh(d, cells, 0.05, False, 2)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                        D.OperatorConfig(d=d, p=p), 0)
    xf = op.quadrature_points("faces")
    fids = op.device_geometry(3).astype(np.int64)
    ref = w.geometry("face_qpoints").reshape(-1, (p + 1) ** (d - 1), d)[fids]
    assert np.array_equal(xf, ref)
    bnd = op.quadrature_points("boundary")
    assert np.array_equal(bnd, faces["exterior_cell"][fids] == D.INVALID_CELL)


def _l2_error(op, x, basis, p, d):
    """|| u_h - u ||_L2 by the k-point Gauss rule (l2_error, bench.cpp:461-520)."""
    from oracle import oracle as O
    from oracle import reflib as R
    S = O.shape_matrices(p, {"lagrange_gauss_lobatto": 0, "lagrange_gauss": 1,
                             "hermite_like": 2}[basis])["S"]
    k = p + 1
    lay = op.layout()
    c = x[: lay.owned_size].reshape((lay.n_owned_cells,) + (k,) * d)
    # canonical index: axis 0 fastest -> numpy axes reversed
    uq = c
    for a in range(d):
        ax = d - a  # numpy axis of the cell-local direction a
        uq = np.moveaxis(np.tensordot(uq, S, axes=([ax], [1])), -1, ax)
    uq = uq.reshape(lay.n_owned_cells, -1)
    xq = op.quadrature_points("cells")
    ue = R.manufactured_solution(d, xq)
    _, wq = O.gauss(k)
    w = wq
    for _ in range(d - 1):
        w = np.multiply.outer(wq, w)
    h = 1.0 / round(lay.n_owned_cells ** (1.0 / d))
    return float(np.sqrt(np.sum((uq - ue) ** 2 * w.reshape(1, -1)) * h ** d))


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_convergence_study(torch, d, p):
    """The reference convergence study (bench.cpp:525-598) on the device:
    make_operator_config's basis, Cartesian unit box, manufactured forcing and
    Dirichlet data through assemble_rhs, device CG to 1e-12; the solution
    matches the reference CG solution of the same system and the L2 error
    converges at order p+1."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    cfg = D.make_operator_config("laplacian", d=d, p=p)
    errs = []
    for level in (1, 2, 3):
        n = 1 << level
        mesh = D.make_box_mesh(d, n, 0.0, False, 1)
        faces = D.enumerate_faces(mesh)
        part = D.partition_cells(mesh, 1)
        D.assign_face_owners(mesh, faces, part)
        op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), cfg, 0)
        xq, xf = op.quadrature_points("cells"), op.quadrature_points("faces")
        f = torch.tensor(R.manufactured_forcing(d, xq).ravel(), device="cuda")
        g = torch.tensor(R.manufactured_solution(d, xf).ravel(), device="cuda")
        b = torch.empty(op.layout().total_size, dtype=torch.float64, device="cuda")
        op.assemble_rhs(b, f, g)
        x = torch.empty_like(b)
        rep = op.conjugate_gradient(b, x, rel_tol=1e-12, max_iterations=100000)
        assert rep["converged"]
        w = R.World(d, [n] * d, p, basis=_RB[cfg.basis], manufactured=True)
        bref = w.rhs(0)
        assert rel_linf(b.cpu().numpy(), bref) < TOL64
        xref, rref = w.cg(bref, 1e-12, 100000)
        assert rref["converged"]
        assert rel_l2(x.cpu().numpy(), xref) < 1e-9
        errs.append(_l2_error(op, x.cpu().numpy(), cfg.basis, p, d))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] > p + 0.5, (errs, rates)


ADV_RANDOM = [
    # d, cells, p, periodic, amplitude, m, ranks, velocity, field, basis
    (3, [3, 3, 2], 1, False, 0.05, 2, 1, (0.85, 0.6, 0.35), 0, "gl"),
    (3, [3, 2, 3], 2, True, 0.04, 2, 2, (-0.3, 0.8, 0.5), 0, "gl"),
    (3, [2, 3, 3], 5, False, 0.05, 2, 3, (0.85, 0.6, 0.35), 0, "gl"),
    (3, [2, 2, 2], 8, False, 0.05, 3, 1, (0.2, -0.7, 0.9), 0, "gl"),
    (2, [6, 5], 7, False, 0.06, 2, 2, (0.85, 0.6, 0.0), 0, "gl"),
    (2, [5, 5], 10, True, 0.03, 2, 1, (0.5, -0.5, 0.0), 0, "gl"),
    (3, [3, 3, 3], 4, False, 0.0, 1, 2, (0.85, 0.6, 0.35), 0, "gl"),
    (3, [3, 3, 2], 3, False, 0.05, 2, 2, (0.0, 0.0, 0.0), 1, "gl"),
    (2, [4, 4], 6, False, 0.05, 2, 1, (0.0, 0.0, 0.0), 1, "gauss"),
    # degenerate meshes: one periodic cell (upwind flux of the cell with
    # itself), one cell per rank (both z neighbours are one ghost cell)
    (3, [1, 1, 1], 3, True, 0.0, 1, 1, (0.85, 0.6, 0.35), 0, "gl"),
    (3, [1, 1, 2], 4, True, 0.0, 1, 2, (-0.3, 0.8, 0.5), 0, "gl"),
    (2, [1, 1], 5, False, 0.0, 1, 1, (0.5, -0.5, 0.0), 0, "gl"),
]


@pytest.mark.parametrize("cfg", ADV_RANDOM, ids=lambda c: f"d{c[0]}p{c[2]}r{c[6]}f{c[8]}-{c[9]}")
def test_advection_against_reference(torch, cfg):
    """The advection apply (OperatorKind::advection, operators.cpp:634-667,
    942-960, 1033-1060) against the reference RankOperator on the same
    inputs; multi-rank cases ship only the planned one-layer ghost values."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p, periodic, amp, m, nr, vel, field, basis = cfg
    w = R.World(d, cells, p, n_ranks=nr, amplitude=amp, mapping_degree=m, periodic=periodic,
                basis=basis, kind="advection", velocity=vel, velocity_field=field)
    x = R.random_vector(w.n_dofs, 2000 + p)
    y_ref = w.apply(x)
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, nr)
    D.assign_face_owners(mesh, faces, part)
    cfg_ = D.OperatorConfig(d=d, p=p, kind="advection", velocity=vel,
                            variable_velocity=bool(field),
                            basis={"gl": "lagrange_gauss_lobatto", "gauss": "lagrange_gauss"}[basis])
    ops = []
    for r in range(nr):
        op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), cfg_, r)
        if field:
            set_field_velocity(op, d)
        ops.append(op)
    if nr == 1:
        y = apply_single(torch, ops[0], x)
    else:
        y = apply_serial_ranks(torch, ops, None, x, (p + 1) ** d, planned_only=basis == "gl")
    assert rel_linf(y, y_ref) < TOL64 and rel_l2(y, y_ref) < TOL64, (rel_linf(y, y_ref),)


@pytest.mark.parametrize("field", [0, 1])
def test_advection_rhs_against_reference(torch, field):
    """assemble_rhs of the advection operator: forcing c.grad u and the inflow
    data (|c.n| - c.n) g (operators.cpp:1053-1060)."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p, vel = 3, [3, 3, 3], 3, (0.85, 0.6, 0.35)
    w = R.World(d, cells, p, n_ranks=2, amplitude=0.05, mapping_degree=2, kind="advection",
                velocity=vel, velocity_field=field, manufactured=True)
    mesh = D.make_box_mesh(d, cells, 0.05, False, 2)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 2)
    D.assign_face_owners(mesh, faces, part)
    for r in range(2):
        op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"),
                            D.OperatorConfig(d=d, p=p, kind="advection", velocity=vel,
                                             variable_velocity=bool(field)), r)
        xq, xf = op.quadrature_points("cells"), op.quadrature_points("faces")
        if field:
            set_field_velocity(op, d)
            cq = R.test_velocity(d, xq)
        else:
            cq = np.broadcast_to(np.array(vel[:d]), xq.shape)
        fq = np.sum(cq * R.manufactured_gradient(d, xq), axis=-1)
        f = torch.tensor(fq.ravel(), device="cuda")
        g = torch.tensor(R.manufactured_solution(d, xf).ravel(), device="cuda")
        rhs = torch.empty(op.layout().total_size, dtype=torch.float64, device="cuda")
        op.assemble_rhs(rhs, f, g)
        torch.cuda.synchronize()
        ref = w.rhs(r)
        got = rhs.cpu().numpy()
        assert rel_linf(got, ref) < TOL64, rel_linf(got, ref)


G4_CASES = [
    # d, cells, p, amplitude, m, periodic, ranks, basis
    (3, [3, 3, 3], 4, 0.05, 2, False, 1, "lagrange_gauss_lobatto"),
    (3, [3, 2, 4], 5, 0.06, 3, False, 3, "hermite_like"),
    (2, [5, 4], 6, 0.05, 2, True, 2, "lagrange_gauss_lobatto"),
    (3, [4, 3, 3], 3, 0.0, 1, False, 1, "lagrange_gauss_lobatto"),
    (3, [2, 2, 3], 2, 0.04, 2, True, 2, "lagrange_gauss"),
]


@pytest.mark.parametrize("cfg", G4_CASES, ids=lambda c: f"d{c[0]}p{c[2]}r{c[6]}-{c[7]}")
def test_geometry_variant_g4_against_reference(torch, cfg):
    """Geometry variant g4 (the merged coefficient J^{-1}J^{-T} det(J) w per
    point, the paper's G4, geometry.cpp:219-246,370-388): device coefficient
    bitwise equal to the reference precompute_geometry, apply equal to the
    reference RankOperator with g4 at 1e-12."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p, amp, m, periodic, nr, basis = cfg
    w = R.World(d, cells, p, n_ranks=nr, amplitude=amp, mapping_degree=m, periodic=periodic,
                basis=_RB[basis], variant="g4")
    x = R.random_vector(w.n_dofs, 4000 + p)
    y_ref = w.apply(x)
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, nr)
    D.assign_face_owners(mesh, faces, part)
    cfg_ = D.OperatorConfig(d=d, p=p, basis=basis, geometry="g4")
    ops = [D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), cfg_, r) for r in range(nr)]
    if nr == 1:
        ns = d * (d + 1) // 2
        nrec = 1 if amp == 0.0 else (p + 1) ** d
        mine = ops[0].device_geometry(0).reshape(-1, ns, nrec).transpose(0, 2, 1).ravel()
        assert np.array_equal(mine, w.geometry("coeff"))
        y = apply_single(torch, ops[0], x)
    else:
        y = apply_serial_ranks(torch, ops, None, x, (p + 1) ** d,
                               planned_only=basis == "hermite_like")
    assert rel_linf(y, y_ref) < TOL64 and rel_l2(y, y_ref) < TOL64, (rel_linf(y, y_ref),)


def test_geometry_variant_g4_host_arrays(torch):
    """g4 from the reference's GeometryCache arrays (DGX_GEOMETRY_HOST_ARRAYS)."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p = 3, [3, 3, 2], 4
    w = R.World(d, cells, p, amplitude=0.05, mapping_degree=2, variant="g4")
    x = R.random_vector(w.n_dofs, 77)
    mesh = D.make_box_mesh(d, cells, 0.05, False, 2)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    arrays = {k: w.geometry(k) for k in ("coeff", "face_jxw", "face_jni", "face_jne", "penalty")}
    arrays["compressed"] = False
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="host_arrays", arrays=arrays),
                        D.OperatorConfig(d=d, p=p, geometry="g4"), 0)
    y = apply_single(torch, op, x)
    assert rel_linf(y, w.apply(x)) < TOL64


def test_apply_argument_errors(torch):
    """apply's argument checks (operators.cpp:220-222: "apply: vector size
    mismatch" is std::invalid_argument) raise before any launch; the operator
    still applies correctly afterwards."""
    D = dgx()
    from paper_1711_03590_b200 import _lib
    op = big_problem(torch, 3, 2, 3, True, D.Geometry())
    N = op.layout().total_size
    u = torch.rand(N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(u)
    with pytest.raises(_lib.DgxInvalidArgument, match="size mismatch"):
        op.apply(u[:-1], y)
    with pytest.raises(_lib.DgxInvalidArgument, match="size mismatch"):
        op.apply(u, torch.empty(N + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(_lib.DgxInvalidArgument, match="float64"):
        op.apply(u.float(), y)
    with pytest.raises(_lib.DgxInvalidArgument, match="GPU"):
        op.apply(u.cpu(), y)
    with pytest.raises(_lib.DgxInvalidArgument, match="contiguous"):
        op.apply(torch.rand(2 * N, dtype=torch.float64, device="cuda")[::2], y)
    op.apply(u, y)
    y2 = torch.empty_like(u)
    op.apply(u, y2)
    assert torch.equal(y, y2)


GUARD_CASES = ([c for c in RANDOM if c[6] == 1 and (min(c[1]) == 1 or c[2] in (4, 5))]
               + [c for c in RANDOM_BASES if c[6] == 1 and (min(c[1]) == 1 or c[2] in (4, 5, 8))])


@pytest.mark.parametrize("cfg", GUARD_CASES, ids=_cfg_id)
def test_guard_bands(torch, cfg):
    """Out-of-bounds check without a sanitizer: u sits between NaN guard bands
    (any read past either end reaches y as NaN) and y between sentinel bands
    (any write past either end changes them); y must match the oracle."""
    from oracle import oracle as O
    D = dgx()
    d, cells, p, periodic, deform, coef, _ = cfg[:7]
    basis = cfg[7] if len(cfg) > 7 else "lagrange_gauss_lobatto"
    P = O.Problem(d, cells, p, periodic=periodic, deform=deform, coefficient=coef, n_ranks=1,
                  basis=O.BASIS[basis])
    amp = deform[1] if deform and deform[0] == "reference" else 0.0
    m = deform[2] if deform and deform[0] == "reference" else 1
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    geo = (D.Geometry(source="vertex_bump", vertex_bump_eps=deform[1], coefficient="a1" if coef else None)
           if deform and deform[0] == "vertex" else D.Geometry(source="mesh"))
    op = D.RankOperator(mesh, part, faces, geo, D.OperatorConfig(d=d, p=p, basis=basis), 0)
    N = op.layout().total_size
    pad = 4096
    x = O.random_vector(P.n_dofs, 5000 + p)
    ub = torch.full((N + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    yb = torch.full((N + 2 * pad,), 12345.0, dtype=torch.float64, device="cuda")
    ub[pad:pad + N] = torch.from_numpy(x).cuda()
    op.apply(ub[pad:pad + N], yb[pad:pad + N])
    torch.cuda.synchronize()
    assert bool((yb[:pad] == 12345.0).all()) and bool((yb[pad + N:] == 12345.0).all())
    y = yb[pad:pad + N].cpu().numpy()
    assert np.isfinite(y).all()
    y_ref = P.apply(x)
    assert rel_linf(y, y_ref) < TOL64


@pytest.mark.parametrize("shape", [("C3", 64, 4, "vertex"), ("C4", 128, 5, "vertex_a"),
                                   ("C5", 160, 6, "cart")], ids=lambda s: s[0])
def test_guard_bands_full_size(torch, shape, free_hbm):
    """The guard-band check at the bench sizes (production grids of the
    pencil-pair and single-pencil kernels): no read past u, no write past y;
    y equals the unguarded apply bitwise."""
    name, n, p, kind = shape
    D = dgx()
    geo = (D.Geometry(source="vertex_bump", vertex_bump_eps=0.1,
                      coefficient="a1" if kind == "vertex_a" else None)
           if kind.startswith("vertex") else D.Geometry())
    op = big_problem(torch, 3, n, p, False, geo)
    N = op.layout().total_size
    pad = 1 << 16
    g = torch.Generator(device="cuda").manual_seed(9)
    ub = torch.full((N + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    ub[pad:pad + N] = torch.rand(N, dtype=torch.float64, device="cuda", generator=g)
    yb = torch.full((N + 2 * pad,), 12345.0, dtype=torch.float64, device="cuda")
    op.apply(ub[pad:pad + N], yb[pad:pad + N])
    y0 = torch.empty(N, dtype=torch.float64, device="cuda")
    op.apply(ub[pad:pad + N].clone(), y0)
    assert bool((yb[:pad] == 12345.0).all()) and bool((yb[pad + N:] == 12345.0).all())
    assert torch.equal(yb[pad:pad + N], y0)
    assert bool(torch.isfinite(y0).all())
    del op, ub, yb, y0


@pytest.mark.parametrize("cfg", [c for c in ADV_RANDOM if c[6] == 1],
                         ids=lambda c: f"d{c[0]}p{c[2]}f{c[8]}-{c[9]}")
def test_guard_bands_advection(torch, cfg):
    """Guard bands (NaN around u, sentinels around y) for the advection
    kernel; y against the reference RankOperator."""
    from oracle import reflib as R
    if not R.available():
        pytest.skip("reference library not built")
    D = dgx()
    d, cells, p, periodic, amp, m, nr, vel, field, basis = cfg
    w = R.World(d, cells, p, n_ranks=1, amplitude=amp, mapping_degree=m, periodic=periodic,
                basis=basis, kind="advection", velocity=vel, velocity_field=field)
    x = R.random_vector(w.n_dofs, 6000 + p)
    mesh = D.make_box_mesh(d, cells, amp, periodic, m)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    cfg_ = D.OperatorConfig(d=d, p=p, kind="advection", velocity=vel,
                            variable_velocity=bool(field),
                            basis={"gl": "lagrange_gauss_lobatto", "gauss": "lagrange_gauss"}[basis])
    op = D.RankOperator(mesh, part, faces, D.Geometry(source="mesh"), cfg_, 0)
    if field:
        set_field_velocity(op, d)
    N = op.layout().total_size
    pad = 4096
    ub = torch.full((N + 2 * pad,), float("nan"), dtype=torch.float64, device="cuda")
    yb = torch.full((N + 2 * pad,), 12345.0, dtype=torch.float64, device="cuda")
    ub[pad:pad + N] = torch.from_numpy(x).cuda()
    op.apply(ub[pad:pad + N], yb[pad:pad + N])
    torch.cuda.synchronize()
    assert bool((yb[:pad] == 12345.0).all()) and bool((yb[pad + N:] == 12345.0).all())
    y = yb[pad:pad + N].cpu().numpy()
    assert rel_linf(y, w.apply(x)) < TOL64
