"""CPU: the product's C ABI and host logic (no GPU needed).

* libdgx.so loads and exports every symbol include/dgx.h declares;
* mesh topology, partition, face owners, ghost maps and exchange plans are
  bit-exact with the reference (golden fixtures);
* the cell task lists cover every computed face exactly once per side;
* errors map onto the reference's exception classes.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, Case, golden_names, load_golden
import paper_1711_03590_b200 as dgx
from paper_1711_03590_b200 import _lib

NAMES = golden_names()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dgx.h")).read()
    return sorted(set(re.findall(r"^(?:dgx_status|const char \*)\s*(dgx_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert b"sm_100a" in _lib.lib().dgx_version()


def mesh_of(c: Case):
    return dgx.make_box_mesh(c.d, c.cells, c.amplitude, c.periodic, c.m)


@pytest.mark.parametrize("name", NAMES)
def test_topology_bitwise(name):
    c = Case(name)
    mesh = mesh_of(c)
    faces = dgx.enumerate_faces(mesh)
    g = c.g
    assert np.array_equal(faces["interior_cell"], g["face_interior"])
    assert np.array_equal(faces["exterior_cell"], g["face_exterior"])
    assert np.array_equal(faces["interior_face_number"], g["face_fn_int"])
    assert np.array_equal(faces["exterior_face_number"], g["face_fn_ext"])
    part = dgx.partition_cells(mesh, c.n_ranks)
    dgx.assign_face_owners(mesh, faces, part)
    assert np.array_equal(part.cell_owner, g["face_cell_owner"])
    assert np.array_equal(part.face_owner, g["face_face_owner"])


def host_op(c: Case, rank, n_ranks=None, p=None):
    mesh = mesh_of(c)
    faces = dgx.enumerate_faces(mesh)
    part = dgx.partition_cells(mesh, n_ranks or c.n_ranks)
    dgx.assign_face_owners(mesh, faces, part)
    cfg = dgx.OperatorConfig(d=c.d, p=p or c.p, basis=c.basis_name, kind=c.kind,
                             velocity=c.velocity, variable_velocity=bool(c.velocity_field))
    return dgx.RankOperator(mesh, part, faces, dgx.Geometry(), cfg, rank, device=-1), faces, part


@pytest.mark.parametrize("name", NAMES)
def test_layout_and_plans_bitwise(name):
    c = Case(name)
    for r in range(c.n_ranks):
        op, _, _ = host_op(c, r)
        lay = op.layout()
        info = c.g[f"r{r}_info"]
        assert [lay.owned_cell_begin, lay.n_owned_cells, lay.owned_size, lay.total_size] == list(info)
        assert np.array_equal(lay.ghost_global_cells, c.g[f"r{r}_ghosts"])
        assert np.array_equal(lay.ghost_owner, c.g[f"r{r}_ghost_owner"])
        for which in ("send", "recv"):
            plans = op.plans(which)
            nbs = c.g[f"r{r}_{which}_neighbors"]
            assert [nb for nb, _ in plans] == list(nbs)
            for i, ((_, cells), (offs, dofs)) in enumerate(zip(plans, op.plan_dofs(which))):
                assert np.array_equal(cells, c.g[f"r{r}_{which}{i}_cells"])
                key = f"r{r}_{which}{i}_dofs"
                if key in c.g:  # Hermite-like: two layers per coupled face
                    assert np.array_equal(offs, c.g[f"r{r}_{which}{i}_offsets"])
                    assert np.array_equal(dofs, c.g[key])
                else:  # whole cells travel
                    nq = lay.dofs_per_cell
                    assert np.array_equal(offs, np.arange(len(cells) + 1) * nq)
                    assert np.array_equal(dofs, np.tile(np.arange(nq), len(cells)))
        # receive plans concatenated = ghost storage order: NCCL receives land
        # directly in the ghost region
        recv = [cells for _, cells in op.plans("recv")]
        if recv:
            assert np.array_equal(np.concatenate(recv), lay.ghost_global_cells)


def tasks_of(op):
    L = _lib.lib()
    n, ni = C.c_int64(), C.c_int64()
    _lib.check(L.dgx_get_tasks(op._h, C.byref(n), C.byref(ni), None, None, None))
    d = op.config.d
    slot = np.empty(n.value, np.int32)
    geo = np.empty(n.value, np.int32)
    fe = np.empty((n.value, 2 * d, 2), np.int32)
    _lib.check(L.dgx_get_tasks(op._h, None, None, slot.ctypes.data_as(C.c_void_p),
                               geo.ctypes.data_as(C.c_void_p), fe.ctypes.data_as(C.c_void_p)))
    return slot, geo, fe, ni.value


@pytest.mark.parametrize("name", NAMES)
def test_task_lists_cover_faces(name):
    """Every face a rank computes is visited once from each of its sides,
    with consistent side bits; every owned cell has one task with its cell
    integral; every ghost cell one ghost-side task."""
    c = Case(name)
    for r in range(c.n_ranks):
        op, faces, part = host_op(c, r)
        lay = op.layout()
        slot, geo, fe, n_inner = tasks_of(op)
        n_owned = lay.n_owned_cells
        n_ghost = len(lay.ghost_global_cells)
        assert sorted(slot) == list(range(n_owned + n_ghost))
        assert all(geo[i] == slot[i] for i in range(len(slot)) if slot[i] < n_owned)
        assert all(geo[i] == -1 for i in range(len(slot)) if slot[i] >= n_owned)
        my_faces = np.nonzero(part.face_owner == r)[0]
        visits = np.zeros(len(my_faces), np.int64)
        sides = np.zeros((len(my_faces), 2), np.int64)
        for t in range(len(slot)):
            for e in fe[t]:
                if e[0] == -2:
                    continue
                rec, side = e[1] & 0x3FFFFFFF, (e[1] >> 30) & 1
                visits[rec] += 1
                sides[rec, side] += 1
                if t < n_inner:
                    assert e[0] < n_owned  # phase 1 never reads a ghost
        boundary = faces["exterior_cell"][my_faces] == dgx.INVALID_CELL
        assert np.all(visits == np.where(boundary, 1, 2))
        assert np.all(sides[:, 0] == 1)
        assert np.all(sides[:, 1] == np.where(boundary, 0, 1))


def test_random_vector_matches_reference_convention():
    g = load_golden("basics")
    for seed in range(5):
        assert np.array_equal(dgx.random_vector(1000, seed), g[f"rng{seed}"])


def test_error_mapping():
    mesh = dgx.make_box_mesh(2, 3, 0.0, False, 1)
    faces = dgx.enumerate_faces(mesh)
    part = dgx.partition_cells(mesh, 1)
    dgx.assign_face_owners(mesh, faces, part)
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=2, p=0), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=2, p=3, W=3), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument, match="Hermite"):
        dgx.RankOperator(mesh, part, faces, dgx.Geometry(),
                         dgx.OperatorConfig(d=2, p=2, basis="hermite_like"), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.RankOperator(mesh, part, faces, dgx.Geometry(),
                         dgx.OperatorConfig(d=2, p=3, basis="bernstein"), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=3, p=3), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.partition_cells(mesh, 100)  # more ranks than cells (mesh.cpp:137-139)
    op = dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=2, p=3), 0, -1)
    with pytest.raises(dgx.DgxInvalidArgument):
        op.apply(0, 8, stream=0)
    bad = faces.copy()
    bad["interior_cell"][0] = 10 ** 6
    with pytest.raises(dgx.DgxInvalidArgument):
        dgx.RankOperator(mesh, part, bad, dgx.Geometry(), dgx.OperatorConfig(d=2, p=3), 0, -1)


def R_available():
    from oracle import reflib as R
    return R.available()


@pytest.mark.skipif(not R_available(), reason="reference library not built")
@pytest.mark.parametrize("cfg", [(3, [4, 3, 5], 4, 5, False), (2, [7, 6], 6, 4, True),
                                 (3, [3, 3, 3], 3, 2, True)])
def test_hermite_plans_match_reference(cfg):
    """Two-layer exchange plans of the Hermite-like basis against the
    reference's build_exchange_plan on more partitions than the fixtures."""
    from oracle import reflib as R
    d, cells, p, nr, periodic = cfg
    w = R.World(d, cells, p, n_ranks=nr, periodic=periodic, basis="hermite")
    mesh = dgx.make_box_mesh(d, cells, 0.0, periodic, 1)
    faces = dgx.enumerate_faces(mesh)
    part = dgx.partition_cells(mesh, nr)
    dgx.assign_face_owners(mesh, faces, part)
    for r in range(nr):
        op = dgx.RankOperator(mesh, part, faces, dgx.Geometry(),
                              dgx.OperatorConfig(d=d, p=p, basis="hermite_like"), r, -1)
        for which in ("send", "recv"):
            ref = w.plans(r, which)
            mine = op.plans(which)
            assert [nb for nb, _ in mine] == [q["neighbor"] for q in ref]
            for (nb, cells_), (offs, dofs), q in zip(mine, op.plan_dofs(which), ref):
                assert np.array_equal(cells_, q["cells"])
                assert np.array_equal(offs, q["offsets"])
                assert np.array_equal(dofs, q["dofs"])


def test_large_topology_matches_oracle():
    """Bigger partitions than the fixtures: 12x10x9 cells over 7 ranks,
    against the C restatement (itself pinned to the reference)."""
    from oracle import oracle as O
    P = O.Problem(3, [12, 10, 9], 2, periodic=True, n_ranks=7)
    mesh = dgx.make_box_mesh(3, (12, 10, 9), 0.0, True, 1)
    faces = dgx.enumerate_faces(mesh)
    part = dgx.partition_cells(mesh, 7)
    dgx.assign_face_owners(mesh, faces, part)
    assert np.array_equal(part.face_owner, P.face_owner)
    for r in (0, 3, 6):
        op = dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=3, p=2), r, -1)
        assert np.array_equal(op.layout().ghost_global_cells, P.rank_ghosts(r))


@pytest.mark.parametrize("R", [2, 4, 8])
def test_c4_size_topology_matches_reference(R):
    """The multi-GPU maps at the size bench.py --gpus N runs (C4: 128^3,
    Dirichlet) against the reference's own functions, compiled unmodified
    in oracle/_ref: enumerate_faces, partition_cells, assign_face_owners
    (mesh.cpp:70-232), every rank's DoFLayout (build_dof_layout,
    dof_layout.cpp:170-253) and exchange plans (build_exchange_plan,
    ghost_exchange.cpp:100-144). Bit-exact. p = 1 keeps the reference's
    per-cell index lists small; the cell sets do not depend on p."""
    from oracle import reflib as R_
    if not R_.available():
        pytest.skip("oracle/_ref not built")
    n, p = 128, 1
    ref = R_.World.topology(3, [n] * 3, p, R)
    fr = ref.faces()
    mesh = dgx.make_box_mesh(3, [n] * 3, 0.0, False, 1)
    faces = dgx.enumerate_faces(mesh)
    assert np.array_equal(faces["interior_cell"], fr["interior"])
    assert np.array_equal(faces["exterior_cell"], fr["exterior"])
    assert np.array_equal(faces["interior_face_number"], fr["fn_int"])
    assert np.array_equal(faces["exterior_face_number"], fr["fn_ext"])
    part = dgx.partition_cells(mesh, R)
    dgx.assign_face_owners(mesh, faces, part)
    assert np.array_equal(part.cell_owner, fr["cell_owner"])
    assert np.array_equal(part.face_owner, fr["face_owner"])
    for r in range(R):
        op = dgx.RankOperator(mesh, part, faces, dgx.Geometry(), dgx.OperatorConfig(d=3, p=p), r, -1)
        lay, rl = op.layout(), ref.layout(r)
        assert (lay.owned_cell_begin, lay.n_owned_cells, lay.owned_size, lay.total_size) == \
            (rl["owned_cell_begin"], rl["n_owned_cells"], rl["owned_size"], rl["total_size"])
        assert np.array_equal(lay.ghost_global_cells, rl["ghost_cells"])
        assert np.array_equal(lay.ghost_owner, rl["ghost_owner"])
        for which in ("send", "recv"):
            mine, theirs = op.plans(which), ref.plans(r, which)
            assert [nb for nb, _ in mine] == [q["neighbor"] for q in theirs]
            for (nb, cells), (offs, dofs), q in zip(mine, op.plan_dofs(which), theirs):
                assert np.array_equal(cells, q["cells"])
                assert np.array_equal(offs, q["offsets"])
                assert np.array_equal(dofs, q["dofs"])
        del op
