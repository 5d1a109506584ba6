"""ctypes binding of include/dgx.h (libdgx.so, built in-tree for sm_100a).

The product path: every call lands in the CUDA library; there is no CPU
fallback. If libdgx.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DGX_LIB overrides the library path (kernel experiments only)
LIB_PATH = os.environ.get("DGX_LIB") or os.path.join(_HERE, "libdgx.so")


class DgxError(RuntimeError):
    pass


class DgxInvalidArgument(DgxError, ValueError):
    """std::invalid_argument in the reference."""


class DgxLogicError(DgxError):
    """std::logic_error in the reference."""


class DgxRuntimeError(DgxError):
    """std::runtime_error in the reference."""


class DgxCudaError(DgxError):
    pass


_STATUS = {1: DgxInvalidArgument, 2: DgxLogicError, 3: DgxRuntimeError,
           4: DgxCudaError}


class RawFace(C.Structure):
    """dg::RawFace (mesh.hpp:80-93), 12 bytes."""
    _fields_ = [("interior_cell", C.c_uint32), ("exterior_cell", C.c_uint32),
                ("interior_face_number", C.c_uint8),
                ("exterior_face_number", C.c_uint8),
                ("subface_index", C.c_uint8), ("face_orientation", C.c_uint8)]


class CMesh(C.Structure):
    _fields_ = [("d", C.c_int), ("cells_per_dim", C.c_int * 3),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("deform_amplitude", C.c_double), ("mapping_degree", C.c_int),
                ("periodic", C.c_int * 3), ("dirichlet_id", C.c_int * 6)]


class CGeometry(C.Structure):
    _fields_ = [("source", C.c_int), ("coefficient", C.c_int),
                ("vertex_bump_eps", C.c_double),
                ("support_points", C.c_void_p), ("support_degree", C.c_int),
                ("cartesian", C.c_int), ("compressed", C.c_int),
                ("inv_jac_t", C.c_void_p), ("jxw", C.c_void_p),
                ("face_jxw", C.c_void_p), ("face_jni", C.c_void_p),
                ("face_jne", C.c_void_p), ("penalty", C.c_void_p),
                ("face_normal", C.c_void_p), ("coeff", C.c_void_p)]


class CConfig(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("W", C.c_int),
                ("basis", C.c_int), ("geometry_variant", C.c_int),
                ("precision", C.c_int), ("kind", C.c_int), ("velocity", C.c_double * 3),
                ("variable_velocity", C.c_int)]


class CSetup(C.Structure):
    _fields_ = [("mesh", CMesh), ("faces", C.c_void_p), ("n_faces", C.c_int64),
                ("n_ranks", C.c_int), ("cell_owner", C.c_void_p),
                ("rank_cell_range", C.c_void_p), ("face_owner", C.c_void_p),
                ("rank", C.c_int), ("config", CConfig), ("geometry", CGeometry)]


class CLayout(C.Structure):
    _fields_ = [("owned_cell_begin", C.c_int64), ("n_owned_cells", C.c_int64),
                ("n_ghost_cells", C.c_int64), ("dofs_per_cell", C.c_int64),
                ("owned_size", C.c_int64), ("total_size", C.c_int64)]


HOOK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class CHooks(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("start_ghost_update", HOOK_FN),
                ("finish_ghost_update", HOOK_FN), ("compress", HOOK_FN)]


class CStats(C.Structure):
    _fields_ = [("n_tasks_inner", C.c_int64), ("n_tasks_coupled", C.c_int64),
                ("n_faces", C.c_int64), ("kernel_launches_per_apply", C.c_int64),
                ("bytes_vectors", C.c_double),
                ("bytes_cell_geometry", C.c_double),
                ("bytes_face_geometry", C.c_double),
                ("cells_per_cta", C.c_int), ("threads_per_cta", C.c_int),
                ("cartesian", C.c_int)]


class CSolveReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int),
                ("relative_residual", C.c_double)]


_lib = None

# every symbol include/dgx.h declares (checked by the CPU test suite)
EXPORTS = [
    "dgx_last_error", "dgx_version", "dgx_enumerate_faces", "dgx_partition",
    "dgx_create", "dgx_destroy", "dgx_get_layout", "dgx_get_ghost_cells",
    "dgx_get_plan", "dgx_get_plan_dofs", "dgx_apply", "dgx_apply_f32", "dgx_apply_host",
    "dgx_apply_phase", "dgx_accumulate_plan", "dgx_conjugate_gradient",
    "dgx_get_quadrature_points", "dgx_assemble_rhs", "dgx_set_velocity", "dgx_nccl_unique_id",
    "dgx_exchanger_create", "dgx_exchanger_hooks", "dgx_exchanger_destroy",
    "dgx_loopback_create", "dgx_loopback_destroy", "dgx_exchanger_create_loopback",
    "dgx_get_geometry", "dgx_get_tasks", "dgx_get_stats", "dgx_random_uniform",
]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libdgx.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.dgx_last_error.restype = C.c_char_p
        L.dgx_version.restype = C.c_char_p
        for name in EXPORTS:
            fn = getattr(L, name)
            if name not in ("dgx_last_error", "dgx_version"):
                fn.restype = C.c_int
        _lib = L
    return _lib


def check(status):
    if status != 0:
        exc = _STATUS.get(status, DgxError)
        raise exc(lib().dgx_last_error().decode())
