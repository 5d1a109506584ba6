"""B200-native matrix-free SIPG-Laplacian apply (arXiv 1711.03590 path).

The package is a thin Python mirror of the reference operator API over the
C ABI of libdgx.so (include/dgx.h): C++ host setup plus hand-written CUDA
kernels for sm_100a. There is no CPU fallback.
"""
from ._lib import (DgxCudaError, DgxError, DgxInvalidArgument, DgxLogicError,
                   DgxRuntimeError)
from .operators import (BASIS_KINDS, FACE_DTYPE, INVALID_CELL, DoFLayout, Geometry,
                        LoopbackExchanger, LoopbackWorld, Mesh, NcclExchanger, OperatorConfig, Partition, RankOperator,
                        assign_face_owners, enumerate_faces, make_box_mesh,
                        make_operator_config, nccl_unique_id, partition_cells, random_vector)

__all__ = [
    "DgxCudaError", "DgxError", "DgxInvalidArgument", "DgxLogicError",
    "DgxRuntimeError", "BASIS_KINDS", "FACE_DTYPE", "INVALID_CELL", "DoFLayout", "Geometry",
    "LoopbackExchanger", "LoopbackWorld", "Mesh", "NcclExchanger", "OperatorConfig", "Partition", "RankOperator",
    "assign_face_owners", "enumerate_faces", "make_box_mesh", "make_operator_config", "nccl_unique_id",
    "partition_cells", "random_vector",
]
