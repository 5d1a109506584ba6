"""Python mirror of the reference operator API for the SIPG-Laplacian path.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/dg/{mesh,operators,dof_layout}.hpp) so that
tests read like the reference's own tests:

    mesh = make_box_mesh(3, 16, 0.0, True, 1)          # mesh.cpp:56-68
    faces = enumerate_faces(mesh)                       # mesh.cpp:70-132
    part = partition_cells(mesh, 1)                     # mesh.cpp:134-155
    assign_face_owners(mesh, faces, part)               # mesh.cpp:157-232
    op = RankOperator(mesh, part, faces, Geometry(), OperatorConfig(d=3, p=3), 0)
    op.apply(u, y)                                      # operators.hpp:85-86

All work happens in libdgx.so (C++ host setup, CUDA kernels for sm_100a).
Vectors are torch CUDA tensors (or raw device pointers) in the reference
rank-local W=1 layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib

FACE_DTYPE = np.dtype([("interior_cell", "<u4"), ("exterior_cell", "<u4"),
                       ("interior_face_number", "u1"),
                       ("exterior_face_number", "u1"),
                       ("subface_index", "u1"), ("face_orientation", "u1")])
assert FACE_DTYPE.itemsize == 12
INVALID_CELL = 0xFFFFFFFF


@dataclass
class Mesh:
    """dg::Mesh (mesh.hpp:24-60)."""
    d: int
    cells_per_dim: tuple
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    deform_amplitude: float = 0.0
    mapping_degree: int = 1
    periodic: tuple = (False, False, False)
    dirichlet_id: tuple = (0, 1, 2, 3, 4, 5)

    def n_cells(self) -> int:
        return int(np.prod(self.cells_per_dim[: self.d]))

    def cartesian(self) -> bool:
        return self.deform_amplitude == 0.0

    def _c(self) -> _lib.CMesh:
        m = _lib.CMesh()
        m.d = self.d
        cells = list(self.cells_per_dim) + [1] * 3
        for a in range(3):
            m.cells_per_dim[a] = int(cells[a]) if a < self.d else 1
            m.lo[a] = float(self.lo[a])
            m.hi[a] = float(self.hi[a])
            m.periodic[a] = int(bool(self.periodic[a]))
        m.deform_amplitude = float(self.deform_amplitude)
        m.mapping_degree = int(self.mapping_degree)
        for s in range(6):
            m.dirichlet_id[s] = int(self.dirichlet_id[s])
        return m


def make_box_mesh(d, cells_per_dim, deform_amplitude, periodic,
                  mapping_degree=3) -> Mesh:
    """make_box_mesh (mesh.cpp:56-68): unit box, all-periodic or all-Dirichlet
    (Dirichlet id = side number). cells_per_dim may also be a tuple."""
    if np.isscalar(cells_per_dim):
        cells = (int(cells_per_dim),) * 3
    else:
        cells = tuple(int(c) for c in cells_per_dim) + (1,) * (3 - len(cells_per_dim))
    return Mesh(d=d, cells_per_dim=cells, deform_amplitude=float(deform_amplitude),
                mapping_degree=max(1, int(mapping_degree)),
                periodic=(bool(periodic),) * 3)


def enumerate_faces(mesh: Mesh) -> np.ndarray:
    """Faces axis by axis, cells lexicographic (mesh.cpp:70-132)."""
    m = mesh._c()
    n = C.c_int64()
    check(lib().dgx_enumerate_faces(C.byref(m), None, C.byref(n)))
    out = np.empty(n.value, FACE_DTYPE)
    check(lib().dgx_enumerate_faces(C.byref(m), out.ctypes.data_as(C.c_void_p),
                                    C.byref(n)))
    return out


@dataclass
class Partition:
    """dg::Partition (mesh.hpp:101-113)."""
    n_ranks: int
    cell_owner: np.ndarray
    rank_cell_range: np.ndarray  # (n_ranks, 2)
    face_owner: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def n_owned_cells(self, rank):
        b, e = self.rank_cell_range[rank]
        return int(e - b)


def _partition(mesh, faces, n_ranks):
    m = mesh._c()
    nc = mesh.n_cells()
    owner = np.empty(nc, np.int32)
    ranges = np.empty(2 * n_ranks, np.int32)
    fo = np.empty(len(faces), np.int32)
    check(lib().dgx_partition(C.byref(m), faces.ctypes.data_as(C.c_void_p),
                              C.c_int64(len(faces)), C.c_int(n_ranks),
                              owner.ctypes.data_as(C.c_void_p),
                              ranges.ctypes.data_as(C.c_void_p),
                              fo.ctypes.data_as(C.c_void_p)))
    return owner, ranges.reshape(n_ranks, 2), fo


def partition_cells(mesh: Mesh, n_ranks: int) -> Partition:
    """Contiguous lexicographic slabs, sizes differing by <= 1
    (mesh.cpp:134-155)."""
    owner, ranges, _ = _partition(mesh, enumerate_faces(mesh), n_ranks)
    return Partition(n_ranks, owner, ranges)


def assign_face_owners(mesh: Mesh, faces: np.ndarray, partition: Partition):
    """Face owners (mesh.cpp:157-232), in place."""
    _, _, fo = _partition(mesh, faces, partition.n_ranks)
    partition.face_owner = fo


BASIS_KINDS = {"lagrange_gauss_lobatto": 0, "lagrange_gauss": 1, "hermite_like": 2}


@dataclass
class OperatorConfig:
    """dg::OperatorConfig (operators.hpp:26-51) for this path. basis: one of
    BASIS_KINDS (BasisKind, basis.hpp:10-15); kind: "laplacian" or
    "advection" (with velocity = VelocityField::constant, or
    variable_velocity=True and per-point values through set_velocity)."""
    d: int = 3
    p: int = 3
    W: int = 1
    kind: str = "laplacian"
    basis: str = "lagrange_gauss_lobatto"
    geometry: str = "g3"
    precision: str = "fp64"
    velocity: tuple = (1.0, 1.0, 1.0)
    variable_velocity: bool = False

    def k(self):
        return self.p + 1


def make_operator_config(kind="laplacian", d=3, p=3, W=1, geometry="g3",
                         precision="fp64") -> OperatorConfig:
    """make_operator_config (operators.cpp:27-41): the Laplacian at p >= 3
    uses the Hermite-like basis, everything else the nodal Gauss-Lobatto one."""
    basis = "hermite_like" if kind == "laplacian" and p >= 3 else "lagrange_gauss_lobatto"
    return OperatorConfig(d=d, p=p, W=W, kind=kind, basis=basis, geometry=geometry,
                          precision=precision)


@dataclass
class Geometry:
    """Where the g3 geometry comes from (the reference passes a
    GeometryCache, geometry.hpp:94-147)."""
    source: str = "mesh"  # mesh | vertex_bump | support | host_arrays
    coefficient: Optional[str] = None  # None | "a(x)=1+0.5sin(pi x)cos(pi y)"
    vertex_bump_eps: float = 0.1
    support_points: Optional[np.ndarray] = None
    support_degree: int = 1
    cartesian: bool = False
    arrays: Optional[dict] = None  # reference GeometryCache arrays


_SOURCES = {"mesh": 0, "vertex_bump": 1, "support": 2, "host_arrays": 3}


@dataclass
class DoFLayout:
    """dg::DoFLayout (dof_layout.hpp:110-155), W = 1."""
    rank: int
    owned_cell_begin: int
    n_owned_cells: int
    dofs_per_cell: int
    owned_size: int
    total_size: int
    ghost_global_cells: np.ndarray
    ghost_owner: np.ndarray


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if hasattr(x, "data_ptr"):
        if not x.is_cuda:
            raise _lib.DgxInvalidArgument("apply: vectors must live on the GPU")
        if not x.is_contiguous():
            raise _lib.DgxInvalidArgument("apply: vectors must be contiguous")
        return C.c_void_p(x.data_ptr())
    raise TypeError(f"cannot pass {type(x)} as a device pointer")


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class RankOperator:
    """dg::RankOperator (operators.hpp:69-106) on one B200."""

    def __init__(self, mesh: Mesh, partition: Partition, faces: np.ndarray,
                 geometry: Geometry, config: OperatorConfig, rank: int = 0,
                 device: int = 0):
        if config.kind not in ("laplacian", "advection"):
            raise _lib.DgxInvalidArgument(f"RankOperator: unknown operator {config.kind!r}")
        if config.basis not in BASIS_KINDS:
            raise _lib.DgxInvalidArgument(f"RankOperator: unknown basis {config.basis!r}")
        self.mesh, self.config, self.rank = mesh, config, rank
        faces = np.ascontiguousarray(faces, FACE_DTYPE)
        if len(partition.face_owner) != len(faces):
            assign_face_owners(mesh, faces, partition)
        s = _lib.CSetup()
        s.mesh = mesh._c()
        s.faces = faces.ctypes.data
        s.n_faces = len(faces)
        s.n_ranks = partition.n_ranks
        co = np.ascontiguousarray(partition.cell_owner, np.int32)
        rr = np.ascontiguousarray(partition.rank_cell_range, np.int32).ravel()
        fo = np.ascontiguousarray(partition.face_owner, np.int32)
        s.cell_owner, s.rank_cell_range, s.face_owner = co.ctypes.data, rr.ctypes.data, fo.ctypes.data
        s.rank = rank
        s.config.d, s.config.p, s.config.W = config.d, config.p, config.W
        s.config.basis = BASIS_KINDS[config.basis]
        s.config.geometry_variant = {"g3": 3, "g4": 4}.get(config.geometry, -1)
        s.config.precision = {"fp64": 0, "fp32": 1}[config.precision]
        s.config.kind = 1 if config.kind == "advection" else 0
        for a in range(3):
            s.config.velocity[a] = float(config.velocity[a]) if a < len(config.velocity) else 0.0
        s.config.variable_velocity = int(bool(config.variable_velocity))
        g = s.geometry
        g.source = _SOURCES[geometry.source]
        g.coefficient = 1 if geometry.coefficient else 0
        g.vertex_bump_eps = geometry.vertex_bump_eps
        keep = []
        if geometry.support_points is not None:
            sp = np.ascontiguousarray(geometry.support_points, np.float64)
            keep.append(sp)
            g.support_points = sp.ctypes.data
        g.support_degree = geometry.support_degree
        g.cartesian = int(geometry.cartesian)
        if geometry.arrays is not None:
            a = {k_: np.ascontiguousarray(v, np.float64)
                 for k_, v in geometry.arrays.items() if k_ != "compressed"}
            keep.append(a)
            g.compressed = int(bool(geometry.arrays.get("compressed", False)))
            for name in ("inv_jac_t", "jxw", "face_jxw", "face_jni", "face_jne",
                         "penalty", "face_normal", "coeff"):
                if name in a:
                    setattr(g, name, a[name].ctypes.data)
        h = C.c_void_p()
        check(lib().dgx_create(C.byref(s), C.c_int(device), C.byref(h)))
        self._h = h
        self.device = device
        lay = _lib.CLayout()
        check(lib().dgx_get_layout(h, C.byref(lay)))
        gc = np.empty(lay.n_ghost_cells, np.uint32)
        go = np.empty(lay.n_ghost_cells, np.int32)
        check(lib().dgx_get_ghost_cells(h, gc.ctypes.data_as(C.c_void_p),
                                        go.ctypes.data_as(C.c_void_p)))
        self._layout = DoFLayout(rank, int(lay.owned_cell_begin),
                                 int(lay.n_owned_cells), int(lay.dofs_per_cell),
                                 int(lay.owned_size), int(lay.total_size), gc, go)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.dgx_destroy(h)
            self._h = None

    def layout(self) -> DoFLayout:
        return self._layout

    # -- apply --------------------------------------------------------------
    def apply(self, u, y, hooks=None, stream=None):
        """y = A u (operators.cpp:217-264). u, y: CUDA tensors (float64, or
        float32 for precision='fp32') of layout().total_size values."""
        self._check_vectors(u, y)
        hk = None if hooks is None else C.byref(hooks.c_hooks())
        fn = lib().dgx_apply_f32 if self.config.precision == "fp32" else lib().dgx_apply
        check(fn(self._h, _ptr(u), _ptr(y), hk, _stream(stream)))

    def _check_vectors(self, *vs):
        """Tensor arguments: layout().total_size values of the operator's
        precision ("apply: vector size mismatch", operators.cpp:220-222).
        Raw integer pointers are passed through unchecked, as in the C ABI."""
        want = "torch.float32" if self.config.precision == "fp32" else "torch.float64"
        for v in vs:
            if hasattr(v, "data_ptr"):
                if v.numel() != self._layout.total_size:
                    raise _lib.DgxInvalidArgument("apply: vector size mismatch")
                if str(v.dtype) != want:
                    raise _lib.DgxInvalidArgument(f"apply: {want[6:]} vectors expected")

    def apply_phase(self, phase, u, y, stream=None):
        self._check_vectors(u, y)
        check(lib().dgx_apply_phase(self._h, C.c_int(phase), _ptr(u), _ptr(y),
                                    _stream(stream)))

    def accumulate_plan(self, idx, contrib, y, stream=None):
        check(lib().dgx_accumulate_plan(self._h, C.c_int(idx), _ptr(contrib),
                                        _ptr(y), _stream(stream)))

    def apply_host(self, u, y=None):
        """Host buffers in, host buffer out (dgx_apply_host: single-rank 3D
        layouts pipeline H2D / apply / D2H over z-slabs). u, y: numpy arrays
        or CPU torch tensors (pinned memory lets the copies overlap the
        apply); y is allocated when None. Returns y."""
        def host_ptr(a, what):
            if isinstance(a, np.ndarray):
                if not a.flags.c_contiguous:
                    raise _lib.DgxInvalidArgument(f"apply_host: {what} must be C-contiguous")
                return a.ctypes.data_as(C.c_void_p), a.size, a.dtype == np.float64
            if not hasattr(a, "data_ptr"):
                raise _lib.DgxInvalidArgument(f"apply_host: {what} must be a numpy array or a CPU tensor")
            if getattr(a, "is_cuda", False) or str(getattr(a, "device", "cpu")) != "cpu":
                raise _lib.DgxInvalidArgument(f"apply_host: {what} must be a host (CPU) buffer")
            if not a.is_contiguous():
                raise _lib.DgxInvalidArgument(f"apply_host: {what} must be contiguous")
            return C.c_void_p(a.data_ptr()), a.numel(), str(a.dtype) == "torch.float64"
        if isinstance(u, np.ndarray):
            u = np.ascontiguousarray(u, np.float64)
        if y is None:
            y = np.empty(self._layout.total_size) if isinstance(u, np.ndarray) else u.new_empty(u.shape)
        (pu, nu, okd_u), (py, ny, okd_y) = host_ptr(u, "u"), host_ptr(y, "y")
        if nu != self._layout.total_size or ny != self._layout.total_size:
            raise _lib.DgxInvalidArgument("apply: vector size mismatch")
        if not (okd_u and okd_y):
            raise _lib.DgxInvalidArgument("apply_host: float64 host buffers expected")
        check(lib().dgx_apply_host(self._h, pu, py))
        return y

    def quadrature_points(self, which="cells"):
        """Physical quadrature points: "cells" -> [owned cell, q, d];
        "faces" -> [computed face, qf, d]; "boundary" -> bool per computed
        face (operators.cpp:545-560, 1115-1145)."""
        w = {"cells": 0, "faces": 1, "boundary": 2}[which]
        n = C.c_int64()
        check(lib().dgx_get_quadrature_points(self._h, C.c_int(w), None, C.byref(n)))
        out = np.empty(n.value)
        check(lib().dgx_get_quadrature_points(self._h, C.c_int(w),
                                              out.ctypes.data_as(C.c_void_p), C.byref(n)))
        d = self.config.d
        lay = self._layout
        if w == 0:
            return out.reshape(lay.n_owned_cells, lay.dofs_per_cell, d)
        if w == 1:
            return out.reshape(-1, lay.dofs_per_cell // (self.config.p + 1), d)
        return out.astype(bool)

    def set_velocity(self, c_cells, c_faces, stream=None):
        """Advection with a variable velocity: c at quadrature_points("cells")
        and quadrature_points("faces") (CUDA tensors, [..., d] flattened)."""
        check(lib().dgx_set_velocity(self._h, _ptr(c_cells), _ptr(c_faces), _stream(stream)))

    def assemble_rhs(self, rhs, forcing=None, dirichlet=None, stream=None):
        """RankOperator::assemble_rhs (operators.cpp:266-282). forcing /
        dirichlet: CUDA tensors of f at quadrature_points("cells") and g at
        quadrature_points("faces") (None: zero); rhs: CUDA tensor of
        layout().total_size values, overwritten."""
        check(lib().dgx_assemble_rhs(self._h, _ptr(forcing), _ptr(dirichlet), _ptr(rhs),
                                     _stream(stream)))

    def conjugate_gradient(self, b, x, rel_tol=1e-10, max_iterations=10000, stream=None):
        """conjugate_gradient(make_apply(op), b, x) (solvers.cpp:24-68,189-206)
        on the device; b, x: CUDA tensors of layout().owned_size values.
        Returns dict(converged, iterations, relative_residual)."""
        rep = _lib.CSolveReport()
        check(lib().dgx_conjugate_gradient(self._h, _ptr(b), _ptr(x), C.c_double(rel_tol),
                                           C.c_int(max_iterations), C.byref(rep),
                                           _stream(stream)))
        return {"converged": bool(rep.converged), "iterations": rep.iterations,
                "relative_residual": rep.relative_residual}

    # -- introspection ------------------------------------------------------
    def plans(self, which):
        """Exchange plans (ghost_exchange.hpp:29-52): list of (neighbor, cells)."""
        w = 0 if which == "send" else 1
        n = C.c_int()
        check(lib().dgx_get_plan(self._h, C.c_int(w), C.c_int(-1), C.byref(n),
                                 None, None, None))
        out = []
        for i in range(n.value):
            nb, nc = C.c_int(), C.c_int64()
            check(lib().dgx_get_plan(self._h, C.c_int(w), C.c_int(i), None,
                                     C.byref(nb), C.byref(nc), None))
            cells = np.empty(nc.value, np.uint32)
            check(lib().dgx_get_plan(self._h, C.c_int(w), C.c_int(i), None,
                                     None, None, cells.ctypes.data_as(C.c_void_p)))
            out.append((nb.value, cells))
        return out

    def plan_dofs(self, which):
        """NeighborPlan::dof_offsets / dofs per plan (ghost_exchange.hpp:29-52):
        list of (offsets uint32[n_cells+1], dofs uint32[n_values])."""
        w = 0 if which == "send" else 1
        out = []
        for i in range(len(self.plans(which))):
            nd = C.c_int64()
            check(lib().dgx_get_plan_dofs(self._h, C.c_int(w), C.c_int(i), None,
                                          C.byref(nd), None))
            nc = C.c_int64()
            check(lib().dgx_get_plan(self._h, C.c_int(w), C.c_int(i), None, None,
                                     C.byref(nc), None))
            offs = np.empty(nc.value + 1, np.uint32)
            dofs = np.empty(nd.value, np.uint32)
            check(lib().dgx_get_plan_dofs(self._h, C.c_int(w), C.c_int(i),
                                          offs.ctypes.data_as(C.c_void_p), None,
                                          dofs.ctypes.data_as(C.c_void_p)))
            out.append((offs, dofs))
        return out

    def plan_values(self, which):
        """Flat value indices (slot * k^d + dof) of every plan, in plan order --
        what the transports pack / unpack."""
        lay = self._layout
        nq = lay.dofs_per_cell
        out = []
        for (nb, cells), (offs, dofs) in zip(self.plans(which), self.plan_dofs(which)):
            c = cells.astype(np.int64)
            owned = (c >= lay.owned_cell_begin) & (c < lay.owned_cell_begin + lay.n_owned_cells)
            slots = np.where(owned, c - lay.owned_cell_begin,
                             lay.n_owned_cells + np.searchsorted(lay.ghost_global_cells, c))
            per = np.diff(offs.astype(np.int64))
            out.append((nb, np.repeat(slots, per) * nq + dofs.astype(np.int64)))
        return out

    def device_geometry(self, which):
        n = C.c_int64()
        check(lib().dgx_get_geometry(self._h, C.c_int(which), None, C.byref(n)))
        out = np.empty(n.value)
        check(lib().dgx_get_geometry(self._h, C.c_int(which),
                                     out.ctypes.data_as(C.c_void_p), C.byref(n)))
        return out

    def tasks(self):
        """The device task list in launch order: (slot, geometry record, face
        entries [n_tasks, 2d, 2] = (neighbour slot | -1 boundary | -2 not
        computed, face record | own side << 30), n_inner)."""
        n, ni = C.c_int64(), C.c_int64()
        check(lib().dgx_get_tasks(self._h, C.byref(n), C.byref(ni), None, None, None))
        d = self.config.d
        slot = np.empty(n.value, np.int32)
        geo = np.empty(n.value, np.int32)
        face = np.empty((n.value, 2 * d, 2), np.int32)
        check(lib().dgx_get_tasks(self._h, C.byref(n), C.byref(ni), slot.ctypes.data_as(C.c_void_p),
                                  geo.ctypes.data_as(C.c_void_p), face.ctypes.data_as(C.c_void_p)))
        return slot, geo, face, int(ni.value)

    def stats(self) -> dict:
        st = _lib.CStats()
        check(lib().dgx_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in _lib.CStats._fields_}


class NcclExchanger:
    """GhostExchanger (ghost_exchange.hpp:96-128) over NCCL send/recv."""

    def __init__(self, op: RankOperator, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        check(lib().dgx_exchanger_create(op._h, buf, C.byref(h)))
        self._op = op  # the native exchanger uses the operator in every hook
        self._h = h
        self._hooks = _lib.CHooks()
        check(lib().dgx_exchanger_hooks(h, C.byref(self._hooks)))

    def c_hooks(self):
        return self._hooks

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.dgx_exchanger_destroy(h)
            self._h = None


class LoopbackWorld:
    """In-process transport world for R rank operators (the reference's
    run_ranks + in-process queues, ghost_exchange.cpp:409-430): each rank's
    LoopbackExchanger turns its messages into cudaMemcpyAsync between the
    ranks' device buffers. Run every rank's apply on its own host thread
    (the C calls release the GIL)."""

    def __init__(self, n_ranks: int):
        h = C.c_void_p()
        check(lib().dgx_loopback_create(C.c_int(n_ranks), C.byref(h)))
        self._h = h
        self.n_ranks = n_ranks

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.dgx_loopback_destroy(h)
            self._h = None


class LoopbackExchanger(NcclExchanger):
    """The native device exchanger (the same pack / in-place receive /
    compress / ascending-rank accumulation as NcclExchanger) over the
    in-process loopback transport."""

    def __init__(self, op: RankOperator, world: LoopbackWorld):
        h = C.c_void_p()
        check(lib().dgx_exchanger_create_loopback(op._h, world._h, C.byref(h)))
        self._op = op
        self._world = world  # the transport shares the world's mailboxes
        self._h = h
        self._hooks = _lib.CHooks()
        check(lib().dgx_exchanger_hooks(h, C.byref(self._hooks)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().dgx_nccl_unique_id(buf))
    return buf.raw


def random_vector(n: int, seed: int) -> np.ndarray:
    """std::mt19937(seed) + uniform_real_distribution(-1,1)
    (reference tests/test_helpers.hpp:11-19)."""
    out = np.empty(n, np.float64)
    check(lib().dgx_random_uniform(out.ctypes.data_as(C.c_void_p), C.c_int64(n),
                                   C.c_uint32(seed)))
    return out
