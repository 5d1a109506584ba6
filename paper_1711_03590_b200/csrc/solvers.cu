// Matrix-free conjugate gradients on the device around the SIPG apply:
// the algorithm of the reference conjugate_gradient (solvers.cpp:24-68) with
// the single-rank adaptor make_apply (solvers.cpp:189-206). Vector updates
// are fused (x, r and the new residual norm in one pass) and every reduction
// is a fixed-order two-pass sum, so runs are bitwise repeatable.
#include "operator.hpp"

#include <cmath>

namespace dgx
{
namespace
{
constexpr int kBlocks = 148 * 4;
constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double *sh)
{
  for (int o = 16; o > 0; o >>= 1)
    v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0)
    sh[w] = v;
  __syncthreads();
  v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1)
      v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// partial[b] = sum over block b's grid-stride share of a . b
__global__ void dot_partial(const double *__restrict__ a, const double *__restrict__ b,
                            long long n, double *partial)
{
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0)
    partial[blockIdx.x] = s;
}

// x += alpha p; r -= alpha Ap; partial[b] = block share of r . r
__global__ void update_xr(double *__restrict__ x, double *__restrict__ r,
                          const double *__restrict__ p, const double *__restrict__ ap,
                          long long n, const double *__restrict__ alpha_dev, double *partial)
{
  __shared__ double sh[32];
  const double alpha = *alpha_dev;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    {
      x[i] += alpha * p[i];
      const double ri = r[i] - alpha * ap[i];
      r[i] = ri;
      s += ri * ri;
    }
  s = block_sum(s, sh);
  if (threadIdx.x == 0)
    partial[blockIdx.x] = s;
}

// p = r + beta p
__global__ void update_p(double *__restrict__ p, const double *__restrict__ r, long long n,
                         const double *__restrict__ beta_dev)
{
  const double beta = *beta_dev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * p[i];
}

// out = sum of the partials in block order (one warp, fixed order)
__global__ void finish_sum(const double *partial, int nb, double *out)
{
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32)
    s += partial[i];
  for (int o = 16; o > 0; o >>= 1)
    s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0)
    *out = s;
}
} // namespace

dgx_solve_report conjugate_gradient(Operator &op, const double *b, double *x, double rel_tol,
                                    int max_iterations, cudaStream_t s)
{
  if (!op.layout().ghosts.empty())
    fail(Code::invalid_argument, "make_apply: operator must be single-rank (no ghost cells)");
  if (op.precision() != 0)
    fail(Code::invalid_argument, "conjugate_gradient: fp64 operators only");
  cuda_check(cudaSetDevice(op.device()), "cudaSetDevice");
  const long long n = op.layout().owned_size();
  dgx_solve_report rep{};
  DeviceArray<double> r(n), p(n), ap(n), partial(kBlocks), scal(4);
  // scal: [0] work, [1] alpha, [2] beta
  cuda_check(cudaMemsetAsync(x, 0, n * 8, s), "memset x");
  cuda_check(cudaMemcpyAsync(r.get(), b, n * 8, cudaMemcpyDeviceToDevice, s), "copy");
  cuda_check(cudaMemcpyAsync(p.get(), b, n * 8, cudaMemcpyDeviceToDevice, s), "copy");
  auto dot = [&](const double *a, const double *c) {
    dot_partial<<<kBlocks, kThreads, 0, s>>>(a, c, n, partial.get());
    finish_sum<<<1, 32, 0, s>>>(partial.get(), kBlocks, scal.get());
    double h = 0;
    cuda_check(cudaMemcpyAsync(&h, scal.get(), 8, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return h;
  };
  const double norm_b = std::sqrt(dot(b, b));
  if (norm_b == 0.0)
    {
      rep.converged = 1;
      return rep;
    }
  double rr = dot(r.get(), r.get());
  for (int it = 0; it < max_iterations; ++it)
    {
      op.apply(p.get(), ap.get(), nullptr, s, false);
      const double pap = dot(p.get(), ap.get());
      if (!(pap > 0.0))
        fail(Code::runtime_error, "conjugate_gradient: operator is not positive definite");
      const double alpha = rr / pap;
      cuda_check(cudaMemcpyAsync(scal.get() + 1, &alpha, 8, cudaMemcpyHostToDevice, s), "h2d");
      update_xr<<<kBlocks, kThreads, 0, s>>>(x, r.get(), p.get(), ap.get(), n, scal.get() + 1,
                                             partial.get());
      finish_sum<<<1, 32, 0, s>>>(partial.get(), kBlocks, scal.get());
      double rr_new = 0;
      cuda_check(cudaMemcpyAsync(&rr_new, scal.get(), 8, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "sync");
      rep.iterations = it + 1;
      rep.relative_residual = std::sqrt(rr_new) / norm_b;
      if (rep.relative_residual <= rel_tol)
        {
          rep.converged = 1;
          return rep;
        }
      const double beta = rr_new / rr;
      rr = rr_new;
      cuda_check(cudaMemcpyAsync(scal.get() + 2, &beta, 8, cudaMemcpyHostToDevice, s), "h2d");
      update_p<<<kBlocks, kThreads, 0, s>>>(p.get(), r.get(), n, scal.get() + 2);
    }
  cuda_check(cudaGetLastError(), "cg kernels");
  return rep;
}

} // namespace dgx
