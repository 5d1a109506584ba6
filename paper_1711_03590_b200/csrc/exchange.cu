// Halo pack / unpack / compress kernels. The exchange plans list, per
// neighbour, the cell-local dofs that travel (whole cells for the nodal and
// generic bases, two layers per coupled face for the Hermite-like basis,
// ghost_exchange.cpp:46-144); the operator flattens them into value index
// lists, so pack / unpack / accumulate are plain indexed copies, coalesced
// over consecutive dofs of a cell.
#include "device.hpp"

namespace dgx
{
namespace
{
template <typename T>
__global__ void gather_values_kernel(const T *__restrict__ src, const long long *__restrict__ index,
                                     long long n, T *__restrict__ dst)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[index[i]];
}

template <typename T>
__global__ void scatter_values_kernel(T *__restrict__ dst, const long long *__restrict__ index,
                                      long long n, const T *__restrict__ src)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[index[i]] = src[i];
}

// dst[index] += src for ONE neighbour plan (no repeated index inside a plan);
// callers launch the plans in ascending neighbour rank so the accumulation
// order is fixed (ghost_exchange.cpp:376-395).
template <typename T>
__global__ void scatter_add_values_kernel(T *__restrict__ dst, const long long *__restrict__ index,
                                          long long n, const T *__restrict__ src)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[index[i]] += src[i];
}

// Whole-cell plans (nodal / generic bases: every plan ships complete cells,
// ghost_exchange.cpp:100-144): the plan is a list of cell slots, and value i
// of the packed message is dof i % nq of cell i / nq -- 4 index bytes per
// cell instead of 8 per value; consecutive threads touch consecutive dofs.
template <typename T>
__global__ void gather_cells_kernel(const T *__restrict__ src, const int *__restrict__ slot,
                                    long long n, int nq, T *__restrict__ dst)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    {
      const long long c = i / nq;
      dst[i] = src[(long long)slot[c] * nq + (i - c * nq)];
    }
}

// dst[cells of ONE neighbour plan] += src (no repeated cell inside a plan)
template <typename T>
__global__ void scatter_add_cells_kernel(T *__restrict__ dst, const int *__restrict__ slot,
                                         long long n, int nq, const T *__restrict__ src)
{
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    {
      const long long c = i / nq;
      dst[(long long)slot[c] * nq + (i - c * nq)] += src[i];
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

// axis-aligned affine records (Operator::cart_): count the compressed cell
// records with an off-diagonal J^{-T} entry above 1e-13 of the diagonal and
// the compressed face records with an n.J^{-T} component off the face axis
// above 1e-13 of the axis one (a box mesh's mapping Jacobian carries
// round-off of ~1e-17 there: the sums of +-x_s/4 over the support points)
__global__ void count_non_axis_kernel(int d, const double *__restrict__ cg, long long n_cells,
                                      const double *__restrict__ fg, const signed char *__restrict__ axis,
                                      long long n_faces, unsigned long long *bad)
{
  unsigned long long mine = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_cells + n_faces; i += stride)
    {
      constexpr double tol = 1e-13;
      if (i < n_cells)
        {
          const double *r = cg + i * (d * d + 1);
          double dmax = 0.0;
          for (int a = 0; a < d; ++a)
            dmax = fmax(dmax, fabs(r[a * d + a]));
          for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b)
              if (a != b && !(fabs(r[a * d + b]) <= tol * dmax))
                ++mine;
        }
      else
        {
          const long long f = i - n_cells;
          const double *r = fg + f * (2 * d + 1);
          const double ni = fabs(r[1 + axis[f]]), ne = fabs(r[1 + d + axis[f]]);
          for (int b = 0; b < d; ++b)
            if (b != axis[f] && !(fabs(r[1 + b]) <= tol * ni && fabs(r[1 + d + b]) <= tol * ne))
              ++mine;
        }
    }
  if (mine)
    atomicAdd(bad, mine);
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
void launch_gather_values(const T *src, const long long *index, long long n, T *dst,
                          cudaStream_t s)
{
  if (n <= 0)
    return;
  gather_values_kernel<<<grid_for(n), 256, 0, s>>>(src, index, n, dst);
  cuda_check(cudaGetLastError(), "gather_values");
}

template <typename T>
void launch_scatter_values(T *dst, const long long *index, long long n, const T *src,
                           cudaStream_t s)
{
  if (n <= 0)
    return;
  scatter_values_kernel<<<grid_for(n), 256, 0, s>>>(dst, index, n, src);
  cuda_check(cudaGetLastError(), "scatter_values");
}

template <typename T>
void launch_scatter_add_values(T *dst, const long long *index, long long n, const T *src,
                               cudaStream_t s)
{
  if (n <= 0)
    return;
  scatter_add_values_kernel<<<grid_for(n), 256, 0, s>>>(dst, index, n, src);
  cuda_check(cudaGetLastError(), "scatter_add_values");
}

template <typename T>
void launch_gather_cells(const T *src, const int *slot, long long n_cells, int nq, T *dst,
                         cudaStream_t s)
{
  const long long n = n_cells * nq;
  if (n <= 0)
    return;
  gather_cells_kernel<<<grid_for(n), 256, 0, s>>>(src, slot, n, nq, dst);
  cuda_check(cudaGetLastError(), "gather_cells");
}

template <typename T>
void launch_scatter_add_cells(T *dst, const int *slot, long long n_cells, int nq, const T *src,
                              cudaStream_t s)
{
  const long long n = n_cells * nq;
  if (n <= 0)
    return;
  scatter_add_cells_kernel<<<grid_for(n), 256, 0, s>>>(dst, slot, n, nq, src);
  cuda_check(cudaGetLastError(), "scatter_add_cells");
}

long long count_non_axis_records(int d, const double *cell_geo, long long n_cells, const double *face_geo,
                                 const signed char *face_axis, long long n_faces)
{
  DeviceArray<unsigned long long> bad(1);
  cuda_check(cudaMemset(bad.get(), 0, sizeof(unsigned long long)), "memset");
  if (n_cells + n_faces > 0)
    count_non_axis_kernel<<<grid_for(n_cells + n_faces), 256>>>(d, cell_geo, n_cells, face_geo, face_axis,
                                                                 n_faces, bad.get());
  cuda_check(cudaGetLastError(), "count_non_axis");
  unsigned long long h = 0;
  cuda_check(cudaMemcpy(&h, bad.get(), sizeof h, cudaMemcpyDeviceToHost), "count_non_axis");
  return (long long)h;
}

template <typename Real>
void launch_convert(const double *src, Real *dst, long long n, cudaStream_t s)
{
  if (n <= 0)
    return;
  convert_kernel<Real><<<grid_for(n), 256, 0, s>>>(src, dst, n);
  cuda_check(cudaGetLastError(), "convert");
}

#define DGX_INST(T)                                                                        \
  template void launch_gather_values<T>(const T *, const long long *, long long, T *,     \
                                        cudaStream_t);                                    \
  template void launch_scatter_values<T>(T *, const long long *, long long, const T *,    \
                                         cudaStream_t);                                   \
  template void launch_scatter_add_values<T>(T *, const long long *, long long, const T *, \
                                             cudaStream_t);                               \
  template void launch_gather_cells<T>(const T *, const int *, long long, int, T *,        \
                                       cudaStream_t);                                     \
  template void launch_scatter_add_cells<T>(T *, const int *, long long, int, const T *,   \
                                            cudaStream_t);
DGX_INST(double)
DGX_INST(float)
#undef DGX_INST
template void launch_convert<float>(const double *, float *, long long, cudaStream_t);
template void launch_convert<double>(const double *, double *, long long, cudaStream_t);

} // namespace dgx
