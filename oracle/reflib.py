"""ctypes view of oracle/_ref/libdgref.so -- the UNMODIFIED reference library
(/root/reference/proj/src) compiled by oracle/ref/Makefile.

TEST INFRASTRUCTURE ONLY. Imported by tests/, tests/golden/make_golden.py,
__graft_entry__.smoke() and bench.py's reference / cpu_baseline legs, always
as the checker or the timed CPU baseline, never as the product path.

A World mirrors the reference test fixtures (SingleRankOp, DistWorld,
BenchWorld) with the nodal Gauss-Lobatto basis forced, Laplacian, geometry
variant g3.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libdgref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library not built: {LIB_PATH}")
        L = C.CDLL(LIB_PATH)
        L.dgref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise RuntimeError("reference: " + lib().dgref_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def manufactured_solution(d, x):
    """exact_solution of the reference convergence study (bench.cpp:437-444);
    x: [..., d] physical points."""
    u = np.cos(2.3 * x[..., 0] + 0.4) * np.cos(1.7 * x[..., 1] - 0.2)
    if d == 3:
        u = u * np.cos(1.1 * x[..., 2] + 0.1)
    return u


def manufactured_gradient(d, x):
    """exact_gradient (bench.cpp:446-453), [..., d]."""
    c0, s0 = np.cos(2.3 * x[..., 0] + 0.4), np.sin(2.3 * x[..., 0] + 0.4)
    c1, s1 = np.cos(1.7 * x[..., 1] - 0.2), np.sin(1.7 * x[..., 1] - 0.2)
    if d == 3:
        c2, s2 = np.cos(1.1 * x[..., 2] + 0.1), np.sin(1.1 * x[..., 2] + 0.1)
        return np.stack([-2.3 * s0 * c1 * c2, -1.7 * c0 * s1 * c2, -1.1 * c0 * c1 * s2], -1)
    return np.stack([-2.3 * s0 * c1, -1.7 * c0 * s1], -1)


def test_velocity(d, x):
    """The harness's variable transport field (ref_capi.cpp test_velocity)."""
    c = np.stack([1.0 + 0.3 * np.sin(2.0 * np.pi * x[..., 1]),
                  0.7 + 0.2 * np.cos(2.0 * np.pi * x[..., 0]),
                  0.4 + 0.1 * x[..., 0] * x[..., 1]], -1)
    return c[..., :d]


def manufactured_forcing(d, x):
    """exact_neg_laplacian (bench.cpp:455-459)."""
    lam = 2.3 * 2.3 + 1.7 * 1.7 + (1.1 * 1.1 if d == 3 else 0.0)
    return lam * manufactured_solution(d, x)


def random_vector(n: int, seed: int) -> np.ndarray:
    """std::mt19937(seed) + uniform_real_distribution<double>(-1,1)."""
    out = np.empty(n, np.float64)
    _chk(lib().dgref_random_vector(C.c_longlong(n), C.c_uint(seed), _p(out)))
    return out


def gauss(n: int, lobatto: bool = False):
    p = np.empty(n)
    w = np.empty(n)
    _chk(lib().dgref_gauss(C.c_int(n), C.c_int(int(lobatto)), _p(p), _p(w)))
    return p, w


BASIS = {"lagrange_gauss_lobatto": 0, "gl": 0, "lagrange_gauss": 1, "gauss": 1,
         "hermite_like": 2, "hermite": 2, "default": -1}


class _basis:
    """Select the BasisKind for the worlds / shape matrices made inside."""

    def __init__(self, basis):
        self.kind = BASIS[basis] if isinstance(basis, str) else int(basis)

    def __enter__(self):
        _chk(lib().dgref_set_basis(C.c_int(self.kind)))

    def __exit__(self, *exc):
        lib().dgref_set_basis(C.c_int(0))


def shape_matrices(p: int, basis="gl"):
    with _basis(basis):
        return _shape_matrices(p)


def _shape_matrices(p: int):
    k = p + 1
    S, D, Dco = (np.empty((k, k)) for _ in range(3))
    Sf, Df = np.empty((2, k)), np.empty((2, k))
    _chk(lib().dgref_shape_matrices(C.c_int(p), _p(S), _p(D), _p(Dco),
                                    _p(Sf), _p(Df)))
    return dict(S=S, D=D, Dco=Dco, Sf=Sf, Df=Df)


GEOM_NAMES = ["inv_jac_t", "jxw", "face_jxw", "face_jni", "face_jne",
              "penalty", "cell_volume", "face_normal", "face_qpoints",
              "wq_cell", "wq_face", "coeff"]


class World:
    """Reference mesh + faces + partition + geometry + one RankOperator per
    rank (proj/tests/test_ghost_exchange.cpp:20-50)."""

    def __init__(self, d, cells, p, n_ranks=1, amplitude=0.0,
                 mapping_degree=1, periodic=False, W=1, geometry=None, basis="gl",
                 manufactured=False, kind="laplacian", velocity=(1.0, 1.0, 1.0),
                 velocity_field=0, variant="g3"):
        """manufactured: forcing / Dirichlet data of the reference convergence
        study (bench.cpp:437-560) for rhs(). kind "advection": the transport
        operator with a constant velocity, or velocity_field=1 (the harness's
        variable test field)."""
        _chk(lib().dgref_set_manufactured(C.c_int(int(manufactured))))
        vel = (C.c_double * 3)(*velocity)
        _chk(lib().dgref_set_operator(C.c_int(1 if kind == "advection" else 0), vel,
                                      C.c_int(velocity_field)))
        self.kind = kind
        _chk(lib().dgref_set_variant(C.c_int(4 if variant == "g4" else 3)))
        try:
            with _basis(basis):
                self._create(d, cells, p, n_ranks, amplitude, mapping_degree, periodic, W,
                             geometry)
        finally:
            lib().dgref_set_manufactured(C.c_int(0))
            lib().dgref_set_operator(C.c_int(0), None, C.c_int(0))
            lib().dgref_set_variant(C.c_int(3))

    @classmethod
    def topology(cls, d, cells, p, n_ranks, periodic=False, basis="gl"):
        """Mesh, faces, partition, layouts and exchange plans only (no
        geometry, no operators): the reference's maps at full sizes."""
        self = cls.__new__(cls)
        self.kind = "laplacian"
        cells = list(cells) + [1] * (3 - len(cells))
        cc = (C.c_int * 3)(*cells)
        h = C.c_void_p()
        self.d, self.p, self.k = d, p, p + 1
        with _basis(basis):
            _chk(lib().dgref_topology_create(C.c_int(d), cc, C.c_int(int(periodic)), C.c_int(p),
                                             C.c_int(n_ranks), C.byref(h)))
        self._h = h
        c = (C.c_longlong * 8)()
        _chk(lib().dgref_world_counts(h, c))
        (self.n_cells, self.n_faces, self.n_q_cell, self.n_q_face,
         self.compressed, self.dofs_per_cell, self.n_ranks,
         self.n_dofs) = [int(x) for x in c]
        return self

    def _create(self, d, cells, p, n_ranks, amplitude, mapping_degree, periodic, W,
                geometry):
        cells = list(cells) + [1] * (3 - len(cells))
        cc = (C.c_int * 3)(*cells)
        h = C.c_void_p()
        self.d, self.p, self.k = d, p, p + 1
        if geometry is None:
            _chk(lib().dgref_world_create(
                C.c_int(d), cc, C.c_double(amplitude), C.c_int(mapping_degree),
                C.c_int(int(periodic)), C.c_int(p), C.c_int(n_ranks),
                C.c_int(W), C.byref(h)))
        else:
            g = {k_: np.ascontiguousarray(v, np.float64)
                 for k_, v in geometry.items() if k_ != "compressed"}
            self._keep = g
            _chk(lib().dgref_world_create_ext(
                C.c_int(d), cc, C.c_int(int(periodic)), C.c_int(p),
                C.c_int(n_ranks), C.c_int(W),
                C.c_int(int(geometry.get("compressed", False))),
                _p(g["inv_jac_t"]), _p(g["jxw"]), _p(g["face_jxw"]),
                _p(g["face_jni"]), _p(g["face_jne"]), _p(g["penalty"]),
                C.byref(h)))
        self._h = h
        c = (C.c_longlong * 8)()
        _chk(lib().dgref_world_counts(h, c))
        (self.n_cells, self.n_faces, self.n_q_cell, self.n_q_face,
         self.compressed, self.dofs_per_cell, self.n_ranks,
         self.n_dofs) = [int(x) for x in c]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.dgref_world_destroy(h)
            self._h = None

    def faces(self):
        n, nc = self.n_faces, self.n_cells
        fi = np.empty(n, np.uint32)
        fe = np.empty(n, np.uint32)
        ni = np.empty(n, np.uint8)
        ne = np.empty(n, np.uint8)
        fo = np.empty(n, np.int32)
        co = np.empty(nc, np.int32)
        _chk(lib().dgref_world_faces(self._h, _p(fi), _p(fe), _p(ni), _p(ne),
                                     _p(fo), _p(co)))
        return dict(interior=fi, exterior=fe, fn_int=ni, fn_ext=ne,
                    face_owner=fo, cell_owner=co)

    def geometry(self, name):
        which = GEOM_NAMES.index(name)
        n = C.c_longlong()
        _chk(lib().dgref_world_geometry(self._h, C.c_int(which), None,
                                        C.byref(n)))
        out = np.empty(n.value)
        _chk(lib().dgref_world_geometry(self._h, C.c_int(which), _p(out),
                                        C.byref(n)))
        return out

    def layout(self, rank):
        info = (C.c_longlong * 5)()
        _chk(lib().dgref_world_layout(self._h, C.c_int(rank), info, None,
                                      None))
        ng = int(info[2])
        gc = np.empty(ng, np.uint32)
        go = np.empty(ng, np.int32)
        _chk(lib().dgref_world_layout(self._h, C.c_int(rank), info, _p(gc),
                                      _p(go)))
        return dict(owned_cell_begin=int(info[0]), n_owned_cells=int(info[1]),
                    owned_size=int(info[3]), total_size=int(info[4]),
                    ghost_cells=gc, ghost_owner=go)

    def plans(self, rank, which):
        """which: 'send' or 'recv' -> list of dict(neighbor, cells,
        offsets, dofs)."""
        w = 0 if which == "send" else 1
        sizes = (C.c_longlong * 4)()
        _chk(lib().dgref_world_plan(self._h, C.c_int(rank), C.c_int(w),
                                    C.c_int(-1), None, None, None, None,
                                    sizes))
        out = []
        for i in range(int(sizes[0])):
            _chk(lib().dgref_world_plan(self._h, C.c_int(rank), C.c_int(w),
                                        C.c_int(i), None, None, None, None,
                                        sizes))
            nb = C.c_int()
            cells = np.empty(int(sizes[1]), np.uint32)
            offs = np.empty(int(sizes[2]), np.uint32)
            dofs = np.empty(int(sizes[3]), np.uint32)
            _chk(lib().dgref_world_plan(self._h, C.c_int(rank), C.c_int(w),
                                        C.c_int(i), C.byref(nb), _p(cells),
                                        _p(offs), _p(dofs), sizes))
            out.append(dict(neighbor=nb.value, cells=cells, offsets=offs,
                            dofs=dofs))
        return out

    def apply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        assert x.size == self.n_dofs
        y = np.empty_like(x)
        _chk(lib().dgref_world_apply(self._h, _p(x), _p(y)))
        return y

    def apply_rank_local(self, rank, u_local):
        u_local = np.ascontiguousarray(u_local, np.float64)
        y = np.empty_like(u_local)
        _chk(lib().dgref_world_apply_rank_local(self._h, C.c_int(rank),
                                                _p(u_local), _p(y)))
        return y

    def assemble(self):
        n = self.n_dofs
        a = np.empty((n, n))
        _chk(lib().dgref_world_assemble(self._h, _p(a)))
        return a

    def rhs(self, rank=0):
        """RankOperator::assemble_rhs of one rank, rank-local layout (W=1)."""
        n = self.layout(rank)["total_size"]
        out = np.empty(n)
        _chk(lib().dgref_world_rhs(self._h, C.c_int(rank), _p(out)))
        return out

    def cg(self, b, rel_tol=1e-10, max_iterations=10000):
        """conjugate_gradient(make_apply(op), b, x) of the reference."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        conv, its, res = C.c_int(), C.c_int(), C.c_double()
        _chk(lib().dgref_world_cg(self._h, _p(b), _p(x), C.c_double(rel_tol),
                                  C.c_int(max_iterations), C.byref(conv), C.byref(its),
                                  C.byref(res)))
        return x, dict(converged=bool(conv.value), iterations=its.value,
                       relative_residual=res.value)

    def time(self, n_applies):
        s = C.c_double()
        _chk(lib().dgref_world_time(self._h, C.c_longlong(n_applies),
                                    C.byref(s)))
        return s.value

    def flops(self):
        f = C.c_double()
        _chk(lib().dgref_world_flops(self._h, C.byref(f)))
        return f.value
