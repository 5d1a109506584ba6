"""GPU parity at the BASELINE configurations' full sizes (north_star: rel L2 /
L_inf <= 1e-12 in fp64, 1e-5 in fp32, against the reference's CPU apply).

* C1 (16^3 periodic, p=3, seed 0), C2 (256^2 Dirichlet, p=1..10, seed 1):
  the whole output vector against the live reference RankOperator::apply
  (oracle/_ref: the unmodified reference compiled here), same input buffer.
* C3 (64^3, BASELINE vertex deformation, p=4, seed 2): the whole vector
  against the live reference RankOperator with the g3 geometry injected from
  the C restatement (the BASELINE deformation is not expressible by the
  reference Mesh; the restatement is pinned bitwise to precompute_geometry,
  SURVEY.md s.8c).
* C4 (128^3, a(x) folded, p=5) and C5 (160^3 Cartesian, p=6, fp64 and fp32):
  sampled cells. y on a cell depends only on the cell, its 2d neighbours and
  their geometry, so each sampled cell is checked against the C restatement
  oracle (pinned to the reference) evaluated on its 3x3x3 patch of the full
  mesh -- the same support points (hence the same J^-T, JxW, normals, face
  JxW, cell volumes and penalties, a(x) at the same physical points), the
  same u. The sample (>= 2000 cells) holds the domain corners, edges and
  boundary-adjacent cells, both sides of every 8-row traversal-tile boundary
  in y, the cells at CTA-partner boundaries of the task order, the first and
  last cells (cell-geometry offsets beyond 2^32 doubles at C4), and random
  cells.
"""
import gc

import numpy as np
import pytest

from conftest import rel_l2, rel_linf

pytestmark = pytest.mark.gpu

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
    gc.collect()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    torch.cuda.empty_cache()


def _dgx():
    import paper_1711_03590_b200 as m
    return m


def _ref_available():
    from oracle import reflib as R
    return R.available()


def _op(d, cells, p, periodic, geometry, precision="fp64"):
    D = _dgx()
    mesh = D.make_box_mesh(d, cells, 0.0, periodic, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    return D.RankOperator(mesh, part, faces, geometry, D.OperatorConfig(d=d, p=p, precision=precision))


def _device_apply(torch, op, x, dtype=None):
    dtype = dtype or torch.float64
    u = torch.tensor(x, dtype=dtype, device="cuda")
    y = torch.empty_like(u)
    op.apply(u, y)
    torch.cuda.synchronize()
    return y.double().cpu().numpy()


def test_c1_whole_vector_vs_reference(torch):
    """C1: 16^3 periodic Cartesian, p=3, input U[-1,1] from seed 0."""
    if not _ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle import reflib as R
    d, n, p = 3, 16, 3
    op = _op(d, [n] * d, p, True, _dgx().Geometry())
    x = _dgx().random_vector(n ** d * (p + 1) ** d, 0)
    ref = R.World(d, [n] * d, p, periodic=True, W=4).apply(x)
    y = _device_apply(torch, op, x)
    assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64


@pytest.mark.parametrize("p", list(range(1, 11)))
def test_c2_whole_vector_vs_reference(torch, p):
    """C2: 256^2 Dirichlet Cartesian, p = 1..10, input from seed 1."""
    if not _ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle import reflib as R
    d, n = 2, 256
    op = _op(d, [n] * d, p, False, _dgx().Geometry())
    x = _dgx().random_vector(n ** d * (p + 1) ** d, 1)
    ref = R.World(d, [n] * d, p, W=4).apply(x)
    y = _device_apply(torch, op, x)
    assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64


def test_c3_whole_vector_vs_reference(torch, free_hbm):
    """C3: 64^3 BASELINE vertex deformation, p=4, per-q J^-T and JxW, seed 2;
    the reference RankOperator with the restatement's g3 arrays injected."""
    if not _ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle import oracle as O
    from oracle import reflib as R
    d, n, p = 3, 64, 4
    P = O.Problem(d, [n] * d, p, deform=("vertex", 0.1))
    geo = {k: P.geom[k] for k in ("inv_jac_t", "jxw", "face_jxw", "face_jni", "face_jne", "penalty")}
    geo["compressed"] = False
    w = R.World(d, [n] * d, p, W=4, n_ranks=1, geometry=geo)
    del P
    x = _dgx().random_vector(n ** d * (p + 1) ** d, 2)
    ref = w.apply(x)
    del w, geo
    op = _op(d, [n] * d, p, False, _dgx().Geometry(source="vertex_bump", vertex_bump_eps=0.1))
    y = _device_apply(torch, op, x)
    assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64


# ---- sampled cells at C4 / C5 ------------------------------------------------

def sample_cells(n, op, n_random=1200, seed=7):
    """Cell ids (single rank: slot = cell id) of the full-size sample."""
    rng = np.random.default_rng(seed)
    ids = set()

    def cid(x, y, z):
        return int(x + n * (y + n * z))

    ends = (0, 1, n // 2, n - 2, n - 1)
    for x in ends:  # corners, edges, face centres, boundary-adjacent layers
        for y in ends:
            for z in ends:
                ids.add(cid(x, y, z))
    for _ in range(150):  # both sides of the 8-row traversal tiles in y
        t = 8 * int(rng.integers(1, max(2, n // 8)))
        x, z = (int(v) for v in rng.integers(0, n, 2))
        for y in (t - 1, t):
            if 0 <= y < n:
                ids.add(cid(x, y, z))
    slot, geo, face, n_inner = op.tasks()
    nc = op.stats()["cells_per_cta"]
    b = np.arange(nc, slot.size, nc)
    for j in rng.choice(b.size, size=min(250, b.size), replace=False):
        ids.add(int(slot[b[j] - 1]))  # last task of a CTA and first of the next
        ids.add(int(slot[b[j]]))
    ids.update(range(0, 20))
    ids.update(range(n ** 3 - 60, n ** 3))  # last cells: largest record offsets
    last_layers = n ** 3 - n * n * 6
    ids.update(int(v) for v in rng.integers(last_layers, n ** 3, 200))
    ids.update(int(v) for v in rng.integers(0, n ** 3, n_random))
    return np.array(sorted(ids), np.int64)


def patch_reference(c, n, k, support, u_cells, compress, coefficient):
    """The C restatement on the 3x3x3 patch (clipped at the domain boundary)
    around cell c of the full n^3 mesh: y on c."""
    from oracle import oracle as O
    d = 3
    ijk = [c % n, (c // n) % n, c // (n * n)]
    lo = [max(t - 1, 0) for t in ijk]
    hi = [min(t + 1, n - 1) for t in ijk]
    pc = [h - l + 1 for l, h in zip(lo, hi)]
    gz, gy, gx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1),
                             np.arange(lo[0], hi[0] + 1), indexing="ij")
    ids = (gx + n * (gy + n * gz)).ravel()
    fc = O.faces(d, pc, False)
    geom = O.geometry(d, pc, 1, support[ids].ravel(), k, compress, coefficient, fc)
    if compress:
        # compressed (Cartesian) records take the cell volume from the box and
        # the cell counts, prod (hi - lo) / cells (geometry.cpp:267-275); the
        # patch's own counts would give 1/prod(pc) instead of the full mesh's
        # 1/n^3, and the penalty tau ~ 1/V scales with it
        geom["penalty"] = geom["penalty"] * (n ** 3 / float(np.prod(pc)))
    u = u_cells(ids).ravel()
    y = O.apply_rank(d, k, ids.size, geom, fc, u)
    me = int(np.nonzero(ids == c)[0][0])
    nq = k ** d
    return y[me * nq:(me + 1) * nq]


def check_sampled(torch, n, p, geometry, support, compress, coefficient, precision="fp64", seed=4):
    k, d = p + 1, 3
    nq = k ** d
    op = _op(d, [n] * d, p, False, geometry, precision)
    N = op.layout().total_size
    dt = torch.float32 if precision == "fp32" else torch.float64
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = (torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).to(dt)
    y = torch.empty_like(u)
    op.apply(u, y)
    torch.cuda.synchronize()
    cells = sample_cells(n, op)
    assert cells.size >= 2000
    uc = u.view(-1, nq)
    y_s = y.view(-1, nq)[torch.from_numpy(cells).cuda()].double().cpu().numpy()

    def u_cells(ids):
        return uc[torch.from_numpy(ids).cuda()].double().cpu().numpy()

    # u of every patch cell in one download, then the patches on all host
    # cores (the oracle's C calls release the GIL)
    need = np.unique(np.concatenate([
        (lambda c: np.array([[x, y, z] for z in range(max(c // (n * n) - 1, 0), min(c // (n * n) + 2, n))
                             for y in range(max((c // n) % n - 1, 0), min((c // n) % n + 2, n))
                             for x in range(max(c % n - 1, 0), min(c % n + 2, n))]))(int(c))
        @ np.array([1, n, n * n]) for c in cells]))
    u_need = u_cells(need)
    pos = {int(v): i for i, v in enumerate(need)}

    def u_local(ids):
        return u_need[[pos[int(i)] for i in ids]]

    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        ref = np.stack(list(ex.map(
            lambda c: patch_reference(int(c), n, k, support, u_local, compress, coefficient), cells)))
    del op, u, y
    tol = TOL32 if precision == "fp32" else TOL64
    scale = np.abs(ref).max()
    err = np.abs(y_s - ref).max(axis=1) / scale
    worst = int(np.argmax(err))
    assert err.max() < tol, f"cell {cells[worst]}: rel L_inf {err.max():.3e}"
    assert rel_l2(y_s, ref) < tol
    return cells.size


def test_c4_sampled_cells(torch, free_hbm):
    """C4: 128^3 vertex-deformed, a(x) folded, p=5 (pencil-pair kernel)."""
    from oracle import oracle as O
    n, p = 128, 5
    support = O.support_vertex_bump(3, [n] * 3, 0.1).reshape(n ** 3, 8, 3)
    geo = _dgx().Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1")
    check_sampled(torch, n, p, geo, support, compress=False, coefficient=True)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c5_sampled_cells(torch, free_hbm, precision):
    """C5: 160^3 Cartesian (compressed affine records), p=6, fp64 and fp32."""
    from oracle import oracle as O
    n, p = 160, 6
    support = O.support_reference(3, [n] * 3, 0.0, 1).reshape(n ** 3, 8, 3)
    check_sampled(torch, n, p, _dgx().Geometry(), support, compress=True, coefficient=False,
                  precision=precision)


def test_ny_beyond_one_tile(torch):
    """3D meshes with more than 8 rows in y (the traversal tiles are full
    x-rows x 8 y-rows): 9 x 17 x 4 at p=5 (pair kernel) and p=4 (single
    pencil), deformed, against the C restatement on the whole mesh."""
    from oracle import oracle as O
    D = _dgx()
    cells = [9, 17, 4]
    for p in (5, 4):
        mesh = D.make_box_mesh(3, cells, 0.0, False, 1)
        faces = D.enumerate_faces(mesh)
        part = D.partition_cells(mesh, 1)
        D.assign_face_owners(mesh, faces, part)
        op = D.RankOperator(mesh, part, faces,
                            D.Geometry(source="vertex_bump", vertex_bump_eps=0.1, coefficient="a1"),
                            D.OperatorConfig(d=3, p=p))
        x = D.random_vector(int(np.prod(cells)) * (p + 1) ** 3, 3)
        ref = O.Problem(3, cells, p, deform=("vertex", 0.1), coefficient=True).apply(x)
        y = _device_apply(torch, op, x)
        assert rel_linf(y, ref) < TOL64 and rel_l2(y, ref) < TOL64


@pytest.mark.parametrize("d,cells,p,periodic,basis", [
    (3, [4, 5, 3], 6, False, "lagrange_gauss_lobatto"),   # C5 shape, odd k
    (3, [3, 4, 5], 4, True, "lagrange_gauss_lobatto"),
    (3, [3, 3, 4], 4, False, "hermite_like"),
    (3, [3, 4, 3], 2, False, "lagrange_gauss"),
    (2, [6, 5], 5, False, "lagrange_gauss_lobatto"),
])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cart_kernel(torch, d, cells, p, periodic, basis, precision):
    """Cartesian box meshes run the tensor-product kernel or the
    collocation CART kernels (DGX_NO_TENSOR; axis-aligned
    affine records: the tangential face terms, products with round-off zeros,
    are skipped): flagged in stats, equal to the general kernel (DGX_NO_CART)
    to round-off and to the C restatement within the parity tolerance."""
    import os
    from oracle import oracle as O
    D = _dgx()
    mesh = D.make_box_mesh(d, cells, 0.0, periodic, 1)
    faces = D.enumerate_faces(mesh)
    part = D.partition_cells(mesh, 1)
    D.assign_face_owners(mesh, faces, part)
    cfg = D.OperatorConfig(d=d, p=p, basis=basis, precision=precision)
    op = D.RankOperator(mesh, part, faces, D.Geometry(), cfg)
    os.environ["DGX_NO_CART"] = "1"
    try:
        gen = D.RankOperator(mesh, part, faces, D.Geometry(), cfg)
    finally:
        del os.environ["DGX_NO_CART"]
    os.environ["DGX_NO_TENSOR"] = "1"
    try:
        col = D.RankOperator(mesh, part, faces, D.Geometry(), cfg)
    finally:
        del os.environ["DGX_NO_TENSOR"]
    # the tensor-product kernel (2); DGX_NO_TENSOR: the collocation CART kernels (1)
    assert op.stats()["cartesian"] == 2
    assert col.stats()["cartesian"] == 1 and gen.stats()["cartesian"] == 0
    x = D.random_vector(int(np.prod(cells)) * (p + 1) ** d, 9)
    dt = torch.float32 if precision == "fp32" else torch.float64
    y = _device_apply(torch, op, x, dt)
    yg = _device_apply(torch, gen, x, dt)
    yc = _device_apply(torch, col, x, dt)
    assert rel_linf(yc, yg) < (1e-5 if precision == "fp32" else 1e-13)
    b = {"lagrange_gauss_lobatto": 0, "lagrange_gauss": 1, "hermite_like": 2}[basis]
    ref = O.Problem(d, cells, p, periodic=periodic, basis=b).apply(x)
    tol = TOL32 if precision == "fp32" else TOL64
    assert rel_linf(y, ref) < tol and rel_l2(y, ref) < tol
    assert rel_linf(y, yg) < (1e-5 if precision == "fp32" else 1e-13)
