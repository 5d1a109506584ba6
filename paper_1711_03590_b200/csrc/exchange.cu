// Halo pack / compress kernels. With the Gauss-Lobatto basis and a face
// normal derivative the reference ships whole cells (all k^d dofs,
// ghost_exchange.cpp:49-96), so pack and accumulate are
// cell-granular gathers: one CTA per cell batch, coalesced over dofs.
#include "device.hpp"

namespace dgx
{
namespace
{
template <typename T>
__global__ void gather_cells_kernel(const T *__restrict__ src, const int *__restrict__ slots,
                                    int n_cells, long long nq, T *__restrict__ dst)
{
  const long long n = (long long)n_cells * nq;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    {
      const long long c = i / nq, j = i - c * nq;
      dst[i] = src[(long long)slots[c] * nq + j];
    }
}

// y[slot] += buf, one neighbour at a time: callers launch neighbours in
// ascending rank order so the accumulation order is fixed
// (ghost_exchange.cpp:376-395).
template <typename T>
__global__ void scatter_add_cells_kernel(T *__restrict__ dst, const int *__restrict__ slots,
                                         int n_cells, long long nq, const T *__restrict__ src)
{
  const long long n = (long long)n_cells * nq;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    {
      const long long c = i / nq, j = i - c * nq;
      dst[(long long)slots[c] * nq + j] += src[i];
    }
}

template <typename Real>
__global__ void convert_kernel(const double *__restrict__ src, Real *__restrict__ dst,
                               long long n)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = static_cast<Real>(src[i]);
}

unsigned grid_for(long long n)
{
  long long g = (n + 255) / 256;
  if (g > 148 * 16)
    g = 148 * 16;
  return (unsigned)(g > 0 ? g : 1);
}
} // namespace

template <typename T>
void launch_gather_cells(const T *src, const int *slots, int n_cells, long long nq, T *dst,
                         cudaStream_t s)
{
  if (n_cells <= 0)
    return;
  gather_cells_kernel<<<grid_for((long long)n_cells * nq), 256, 0, s>>>(src, slots, n_cells,
                                                                          nq, dst);
  cuda_check(cudaGetLastError(), "gather_cells");
}

template <typename T>
void launch_scatter_add_cells(T *dst, const int *slots, int n_cells, long long nq, const T *src,
                              cudaStream_t s)
{
  if (n_cells <= 0)
    return;
  scatter_add_cells_kernel<<<grid_for((long long)n_cells * nq), 256, 0, s>>>(dst, slots,
                                                                              n_cells, nq, src);
  cuda_check(cudaGetLastError(), "scatter_add_cells");
}

template <typename Real>
void launch_convert(const double *src, Real *dst, long long n, cudaStream_t s)
{
  if (n <= 0)
    return;
  convert_kernel<Real><<<grid_for(n), 256, 0, s>>>(src, dst, n);
  cuda_check(cudaGetLastError(), "convert");
}
template void launch_gather_cells<double>(const double *, const int *, int, long long,
                                         double *, cudaStream_t);
template void launch_gather_cells<float>(const float *, const int *, int, long long, float *,
                                        cudaStream_t);
template void launch_scatter_add_cells<double>(double *, const int *, int, long long,
                                              const double *, cudaStream_t);
template void launch_scatter_add_cells<float>(float *, const int *, int, long long,
                                             const float *, cudaStream_t);
template void launch_convert<float>(const double *, float *, long long, cudaStream_t);
template void launch_convert<double>(const double *, double *, long long, cudaStream_t);

} // namespace dgx
