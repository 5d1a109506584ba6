"""ctypes view of the C restatement oracle (oracle/_build/libdgoracle.so).

TEST INFRASTRUCTURE ONLY -- the checker for tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg. Never the thing measured or shipped.

`Problem` bundles one configuration the way the reference fixtures do:
mesh -> faces (mesh.cpp:70-132) -> partition + face owners (mesh.cpp:134-232)
-> g3 geometry (geometry.cpp:248-522) -> apply (table-based restatement).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libdgoracle.so")
INVALID = 0xFFFFFFFF
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.dgo_last_error.restype = C.c_char_p
        L.dgo_faces.restype = C.c_int64
        L.dgo_ghosts.restype = C.c_int64
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib().dgo_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _cells(cells):
    cells = list(cells) + [1] * (3 - len(cells))
    return (C.c_int * 3)(*cells)


def random_vector(n, seed):
    out = np.empty(n)
    _chk(lib().dgo_random_vector(C.c_int64(n), C.c_uint32(seed), _p(out)))
    return out


def gauss(n, lobatto=False):
    p, w = np.empty(n), np.empty(n)
    _chk(lib().dgo_gauss(C.c_int(n), C.c_int(int(lobatto)), _p(p), _p(w)))
    return p, w


BASIS = {"lagrange_gauss_lobatto": 0, "gl": 0, "lagrange_gauss": 1, "gauss": 1,
         "hermite_like": 2, "hermite": 2}


def basis_kind(basis, p=None):
    """BasisKind index; "default" = make_operator_config's Laplacian choice
    (operators.cpp:27-41)."""
    if basis == "default":
        return 2 if p is not None and p >= 3 else 0
    return BASIS[basis] if isinstance(basis, str) else int(basis)


def shape_matrices(p, basis="gl"):
    k = p + 1
    S, D, Dco = (np.empty((k, k)) for _ in range(3))
    Sf, Df = np.empty((2, k)), np.empty((2, k))
    _chk(lib().dgo_shape(C.c_int(p), C.c_int(basis_kind(basis, p)), _p(S), _p(D), _p(Dco),
                         _p(Sf), _p(Df)))
    return dict(S=S, D=D, Dco=Dco, Sf=Sf, Df=Df)


def faces(d, cells, periodic):
    cc = _cells(cells)
    n = lib().dgo_faces(C.c_int(d), cc, C.c_int(int(periodic)), None, None,
                        None, None)
    fi, fe = np.empty(n, np.uint32), np.empty(n, np.uint32)
    ni, ne = np.empty(n, np.uint8), np.empty(n, np.uint8)
    lib().dgo_faces(C.c_int(d), cc, C.c_int(int(periodic)), _p(fi), _p(fe),
                    _p(ni), _p(ne))
    return dict(interior=fi, exterior=fe, fn_int=ni, fn_ext=ne)


def partition(n_cells, n_ranks):
    owner = np.empty(n_cells, np.int32)
    ranges = np.empty(2 * n_ranks, np.int32)
    _chk(lib().dgo_partition(C.c_int(n_cells), C.c_int(n_ranks), _p(owner),
                             _p(ranges)))
    return owner, ranges.reshape(n_ranks, 2)


def face_owners(fc, cell_owner):
    n = fc["interior"].size
    fo = np.empty(n, np.int32)
    _chk(lib().dgo_face_owners(C.c_int64(n), _p(fc["interior"]),
                               _p(fc["exterior"]), _p(cell_owner), _p(fo)))
    return fo


def ghosts(rank, fc, face_owner, cell_owner):
    n = fc["interior"].size
    args = (C.c_int(rank), C.c_int64(n), _p(fc["interior"]),
            _p(fc["exterior"]), _p(face_owner), _p(cell_owner))
    ng = lib().dgo_ghosts(*args, None)
    out = np.empty(ng, np.uint32)
    lib().dgo_ghosts(*args, _p(out))
    return out


def support_reference(d, cells, amplitude, m):
    nc = int(np.prod(cells[:d]))
    out = np.empty(nc * (m + 1) ** d * d)
    _chk(lib().dgo_support_reference(C.c_int(d), _cells(cells),
                                     C.c_double(amplitude), C.c_int(m),
                                     _p(out)))
    return out


def support_vertex_bump(d, cells, eps):
    nc = int(np.prod(cells[:d]))
    out = np.empty(nc * 2 ** d * d)
    _chk(lib().dgo_support_vertex_bump(C.c_int(d), _cells(cells),
                                       C.c_double(eps), _p(out)))
    return out


def geometry(d, cells, m, support, k, compress, coefficient, fc):
    nc = int(np.prod(cells[:d]))
    nf = fc["interior"].size
    nq, nqf = k ** d, k ** (d - 1)
    nrec = nc * (1 if compress else nq)
    g = dict(inv_jac_t=np.empty(nrec * d * d), jxw=np.empty(nrec),
             face_jxw=np.empty(nf * nqf), face_jni=np.empty(nf * nqf * d),
             face_jne=np.empty(nf * nqf * d), penalty=np.empty(nf),
             cell_volume=np.empty(nc))
    _chk(lib().dgo_geometry(
        C.c_int(d), _cells(cells), C.c_int(m), _p(np.ascontiguousarray(support)),
        C.c_int(k), C.c_int(int(compress)), C.c_int(int(coefficient)),
        C.c_int64(nf), _p(fc["interior"]), _p(fc["exterior"]),
        _p(fc["fn_int"]), _p(fc["fn_ext"]), _p(g["inv_jac_t"]), _p(g["jxw"]),
        _p(g["face_jxw"]), _p(g["face_jni"]), _p(g["face_jne"]),
        _p(g["penalty"]), _p(g["cell_volume"])))
    g["compressed"] = bool(compress)
    return g


def apply_rank(d, k, n_cells, geom, fc, u, rank=0, face_owner=None,
               cell_range=None, ghost_cells=None, basis=0):
    if cell_range is None:
        cell_range = (0, n_cells)
    gh = (np.zeros(0, np.uint32) if ghost_cells is None
          else np.ascontiguousarray(ghost_cells, np.uint32))
    u = np.ascontiguousarray(u, np.float64)
    y = np.empty_like(u)
    fo = None if face_owner is None else np.ascontiguousarray(face_owner, np.int32)
    _chk(lib().dgo_apply_rank(
        C.c_int(d), C.c_int(k), C.c_int(n_cells),
        C.c_int(int(geom["compressed"])), _p(geom["inv_jac_t"]),
        _p(geom["jxw"]), C.c_int64(fc["interior"].size), _p(fc["interior"]),
        _p(fc["exterior"]), _p(fc["fn_int"]), _p(fc["fn_ext"]),
        _p(geom["face_jxw"]), _p(geom["face_jni"]), _p(geom["face_jne"]),
        _p(geom["penalty"]), C.c_int(rank), _p(fo), C.c_int(cell_range[0]),
        C.c_int(cell_range[1]), C.c_int64(gh.size), _p(gh), _p(u), _p(y), C.c_int(basis)))
    return y


class Problem:
    """One configuration: box mesh (unit cube), basis of degree p (GL unless
    basis= selects lagrange_gauss / hermite_like / default), g3.

    deform: ("reference", amplitude, m) -> Mesh::map_point deformation of the
            reference (mesh.cpp:11-26); ("vertex", eps) -> BASELINE vertex
            bump (trilinear); None -> Cartesian (compressed storage).
    """

    def __init__(self, d, cells, p, periodic=False, deform=None,
                 coefficient=False, n_ranks=1, basis="gl"):
        self.d, self.p, self.k = d, p, p + 1
        self.basis = basis_kind(basis, p)
        self.cells = list(cells)[:d]
        self.n_cells = int(np.prod(self.cells))
        self.periodic = periodic
        self.fc = faces(d, self.cells, periodic)
        self.cell_owner, self.ranges = partition(self.n_cells, n_ranks)
        self.face_owner = face_owners(self.fc, self.cell_owner)
        self.n_ranks = n_ranks
        compress = deform is None and not coefficient
        if deform is None:
            self.m = 1
            sup = support_reference(d, self.cells, 0.0, 1)
        elif deform[0] == "reference":
            self.m = deform[2]
            sup = support_reference(d, self.cells, deform[1], deform[2])
        elif deform[0] == "vertex":
            self.m = 1
            sup = support_vertex_bump(d, self.cells, deform[1])
        else:
            raise ValueError(deform)
        self.support = sup
        self.geom = geometry(d, self.cells, self.m, sup, self.k, compress,
                             coefficient, self.fc)
        self.dofs_per_cell = self.k ** d
        self.n_dofs = self.n_cells * self.dofs_per_cell

    def apply(self, x):
        return apply_rank(self.d, self.k, self.n_cells, self.geom, self.fc, x,
                          basis=self.basis)

    def rank_ghosts(self, rank):
        return ghosts(rank, self.fc, self.face_owner, self.cell_owner)

    def apply_rank_local(self, rank, u_local):
        b, e = self.ranges[rank]
        return apply_rank(self.d, self.k, self.n_cells, self.geom, self.fc,
                          u_local, rank=rank, face_owner=self.face_owner,
                          cell_range=(int(b), int(e)),
                          ghost_cells=self.rank_ghosts(rank), basis=self.basis)
