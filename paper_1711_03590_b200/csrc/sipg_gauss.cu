// Fused SIPG apply kernels for the Lagrange-Gauss (collocation) basis.
#define DGX_BASIS 1
#define DGX_FN(name) name##_gauss
#include "sipg_launch.cuh"
