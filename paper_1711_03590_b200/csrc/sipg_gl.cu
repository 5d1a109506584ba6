// Fused SIPG apply kernels for the nodal Gauss-Lobatto basis.
#define DGX_BASIS 0
#define DGX_FN(name) name##_gl
#include "sipg_launch.cuh"
