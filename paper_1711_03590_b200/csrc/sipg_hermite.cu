// Fused SIPG apply kernels for the Hermite-like basis.
#define DGX_BASIS 2
#define DGX_FN(name) name##_hermite
#include "sipg_launch.cuh"
