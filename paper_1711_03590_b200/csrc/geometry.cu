// Device precompute of the g3 geometry (inverse Jacobian transpose and JxW
// per cell quadrature point; JxW_f, n.J^{-T} of both sides and the penalty
// per face) from mapping support points. Restates the algebra of the
// reference precompute_geometry (geometry.cpp:248-522) with
// mapping_point_jacobian (:65-116) and invert_jacobian (:118-150), but runs
// one thread per (cell, q) / per face on the GPU and writes the SoA layout
// the apply kernel reads (coalesced over q).
//
// Compiled with --fmad=false so the arithmetic reproduces the reference
// (built with -ffp-contract=off) bit for bit on reference meshes.
#include "device.hpp"

namespace dgx
{
namespace
{

struct GeoConst
{
  double qp[16], qw[16]; // Gauss points / weights on [0,1], k <= 11
  double nodes[16];      // Gauss-Lobatto nodes of the mapping degree m
};

__device__ double lag_value(const double *x, int n, int j, double t)
{
  double v = 1.0;
  for (int m = 0; m < n; ++m)
    if (m != j)
      v *= (t - x[m]) / (x[j] - x[m]);
  return v;
}

__device__ double lag_derivative(const double *x, int n, int j, double t)
{
  double sum = 0.0;
  for (int i = 0; i < n; ++i)
    {
      if (i == j)
        continue;
      double v = 1.0 / (x[j] - x[i]);
      for (int m = 0; m < n; ++m)
        if (m != j && m != i)
          v *= (t - x[m]) / (x[j] - x[m]);
      sum += v;
    }
  return sum;
}

// mapping_point_jacobian (geometry.cpp:65-116)
__device__ void map_point_jac(const GeoConst &gc, int d, int n, const double *sp,
                              const double *xi, double *x_out, double *jac)
{
  double val[3][16], der[3][16];
  for (int a = 0; a < d; ++a)
    for (int j = 0; j < n; ++j)
      {
        val[a][j] = lag_value(gc.nodes, n, j, xi[a]);
        der[a][j] = lag_derivative(gc.nodes, n, j, xi[a]);
      }
  for (int i = 0; i < d; ++i)
    x_out[i] = 0.0;
  for (int i = 0; i < d * d; ++i)
    jac[i] = 0.0;
  int np = 1;
  for (int a = 0; a < d; ++a)
    np *= n;
  for (int s = 0; s < np; ++s)
    {
      double shape = 1.0, dshape[3];
      int idx = s, loc[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a)
        {
          loc[a] = idx % n;
          idx /= n;
          shape *= val[a][loc[a]];
        }
      for (int a = 0; a < d; ++a)
        {
          double p = der[a][loc[a]];
          for (int b = 0; b < d; ++b)
            if (b != a)
              p *= val[b][loc[b]];
          dshape[a] = p;
        }
      const double *xs = sp + s * d;
      for (int i = 0; i < d; ++i)
        x_out[i] += shape * xs[i];
      for (int i = 0; i < d; ++i)
        for (int a = 0; a < d; ++a)
          jac[i * d + a] += dshape[a] * xs[i];
    }
}

// invert_jacobian (geometry.cpp:118-150): returns det, writes J^{-T}
__device__ double invert_jac(int d, const double *j, double *jit)
{
  if (d == 2)
    {
      const double det = j[0] * j[3] - j[1] * j[2];
      const double inv = 1.0 / det;
      jit[0] = j[3] * inv;
      jit[1] = -j[2] * inv;
      jit[2] = -j[1] * inv;
      jit[3] = j[0] * inv;
      return det;
    }
  double cof[9];
  cof[0] = j[4] * j[8] - j[5] * j[7];
  cof[1] = j[5] * j[6] - j[3] * j[8];
  cof[2] = j[3] * j[7] - j[4] * j[6];
  cof[3] = j[2] * j[7] - j[1] * j[8];
  cof[4] = j[0] * j[8] - j[2] * j[6];
  cof[5] = j[1] * j[6] - j[0] * j[7];
  cof[6] = j[1] * j[5] - j[2] * j[4];
  cof[7] = j[2] * j[3] - j[0] * j[5];
  cof[8] = j[0] * j[4] - j[1] * j[3];
  const double det = j[0] * cof[0] + j[1] * cof[1] + j[2] * cof[2];
  const double inv = 1.0 / det;
  for (int i = 0; i < 9; ++i)
    jit[i] = cof[i] * inv;
  return det;
}

__device__ double coef_a(const double *x)
{
  return 1.0 + 0.5 * sin(M_PI * x[0]) * cos(M_PI * x[1]);
}

__device__ double cell_weight(const GeoConst &gc, int d, int k, int q)
{
  double w = 1.0;
  for (int a = 0; a < d; ++a)
    {
      w *= gc.qw[q % k];
      q /= k;
    }
  return w;
}

__global__ void cell_geometry_kernel(GeometryJob job, GeoConst gc, int *bad)
{
  const int d = job.d, k = job.k, n = job.m + 1;
  int nq = 1, pp = 1;
  for (int a = 0; a < d; ++a)
    {
      nq *= k;
      pp *= n;
    }
  const long long nrec = job.compress ? 1 : nq;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)job.n_geo_cells * nrec)
    return;
  const int c = (int)(gid / nrec);
  const int rec = (int)(gid - (long long)c * nrec);
  double xi[3] = {0.5, 0.5, 0.5};
  if (!job.compress)
    {
      int idx = rec;
      for (int a = 0; a < d; ++a)
        {
          xi[a] = gc.qp[idx % k];
          idx /= k;
        }
    }
  double x[3], jac[9], jit[9];
  map_point_jac(gc, d, n, job.support + (long long)c * pp * d, xi, x, jac);
  const double det = invert_jac(d, jac, jit);
  if (!(det > 0.0))
    atomicExch(bad, 1);
  double det_jxw = job.compress ? det : det * cell_weight(gc, d, k, rec);
  if (job.coefficient)
    det_jxw *= coef_a(x);
  if (job.g4)
    {
      // symmetric_coefficient (geometry.cpp:219-246): (J^{-1} J^{-T})_ij
      // det(J) w, entries (00, 11, 22, 01, 02, 12) / (00, 11, 01)
      const int ns = d * (d + 1) / 2;
      const int ii[6] = {0, 1, d == 3 ? 2 : 0, 0, 0, 1};
      const int jj[6] = {0, 1, d == 3 ? 2 : 1, 1, 2, 2};
      double *out = job.cell_geo + (long long)c * ns * nrec + rec;
      for (int e = 0; e < ns; ++e)
        {
          const int i = d == 3 ? ii[e] : (e < 2 ? e : 0), j = d == 3 ? jj[e] : (e < 2 ? e : 1);
          double sum = 0;
          for (int a = 0; a < d; ++a)
            sum += jit[a * d + i] * jit[a * d + j];
          out[e * nrec] = sum * det_jxw;
        }
      return;
    }
  const int nc = d * d + 1;
  double *out = job.cell_geo + (long long)c * nc * nrec + rec;
  for (int i = 0; i < d * d; ++i)
    out[i * nrec] = jit[i];
  out[d * d * nrec] = det_jxw;
}

__global__ void volume_kernel(GeometryJob job, GeoConst gc, int *bad)
{
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= job.n_slots)
    return;
  if (job.cart_volume > 0.0) // Cartesian mesh: product of the extents (geometry.cpp:401-407)
    {
      job.volume[slot] = job.cart_volume;
      return;
    }
  const int d = job.d, k = job.k, n = job.m + 1;
  int nq = 1, pp = 1;
  for (int a = 0; a < d; ++a)
    {
      nq *= k;
      pp *= n;
    }
  double v = 0.0;
  for (int q = 0; q < nq; ++q)
    {
      double xi[3] = {0, 0, 0};
      int idx = q;
      for (int a = 0; a < d; ++a)
        {
          xi[a] = gc.qp[idx % k];
          idx /= k;
        }
      double x[3], jac[9], jit[9];
      map_point_jac(gc, d, n, job.support + (long long)slot * pp * d, xi, x, jac);
      const double det = invert_jac(d, jac, jit);
      if (!(det > 0.0))
        atomicExch(bad, 1);
      v += det * cell_weight(gc, d, k, q);
    }
  job.volume[slot] = v;
}

__global__ void face_geometry_kernel(GeometryJob job, GeoConst gc, int *bad)
{
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= job.n_faces)
    return;
  const int d = job.d, k = job.k, n = job.m + 1;
  int nqf = 1, pp = 1;
  for (int a = 0; a < d - 1; ++a)
    nqf *= k;
  for (int a = 0; a < d; ++a)
    pp *= n;
  const int4 fc = job.faces[f];
  const int axis = fc.z / 2;
  int tang[2] = {0, 0}, nt = 0;
  for (int a = 0; a < d; ++a)
    if (a != axis)
      tang[nt++] = a;
  const bool boundary = fc.y < 0;
  // full records [2d+1][nqf]; Cartesian (compressed) records [2d+1][1] hold
  // det |J^{-T} e_axis| without the weight (applied on the fly like the
  // compressed cell records, geometry.hpp:133-143) and the constant normals
  const int nrf = job.compress ? 1 : nqf;
  double *fg = job.face_geo + f * (2 * d + 1) * nrf;
  double area = 0.0, abar = 0.0;
  for (int q = 0; q < nqf; ++q)
    {
      double tc[2] = {0.5, 0.5};
      int idx = q;
      for (int t = 0; t < nt; ++t)
        {
          tc[t] = gc.qp[idx % k];
          idx /= k;
        }
      double wqf = 1.0;
      idx = q;
      for (int a = 0; a < d - 1; ++a)
        {
          wqf *= gc.qw[idx % k];
          idx /= k;
        }
      double xi[3] = {0, 0, 0};
      for (int t = 0; t < nt; ++t)
        xi[tang[t]] = tc[t];
      xi[axis] = fc.z % 2 ? 1.0 : 0.0;
      double xq[3], jac[9], jit[9];
      map_point_jac(gc, d, n, job.support + (long long)fc.x * pp * d, xi, xq, jac);
      const double det = invert_jac(d, jac, jit);
      if (!(det > 0.0))
        atomicExch(bad, 1);
      const double sign = fc.z % 2 ? 1.0 : -1.0;
      double nvec[3], nrm = 0, normal[3];
      for (int i = 0; i < d; ++i)
        {
          nvec[i] = jit[i * d + axis];
          nrm += nvec[i] * nvec[i];
        }
      nrm = sqrt(nrm);
      for (int i = 0; i < d; ++i)
        normal[i] = sign * nvec[i] / nrm;
      if (job.face_normal && (!job.compress || q == 0))
        for (int i = 0; i < d; ++i)
          job.face_normal[(f * d + i) * nrf + q] = normal[i];
      const double jxw_f = det * nrm * wqf;
      if (!job.compress)
        fg[q] = jxw_f;
      else if (q == 0)
        fg[0] = det * nrm;
      area += jxw_f;
      const double a = job.coefficient ? coef_a(xq) : 1.0;
      abar += a;
      double jni[3];
      for (int j = 0; j < d; ++j)
        {
          double s = 0;
          for (int i = 0; i < d; ++i)
            s += normal[i] * jit[i * d + j];
          jni[j] = s;
        }
      double jne[3] = {jni[0], jni[1], jni[2]};
      if (!boundary)
        {
          double xie[3] = {0, 0, 0};
          for (int t = 0; t < nt; ++t)
            xie[tang[t]] = tc[t];
          xie[axis] = fc.w % 2 ? 1.0 : 0.0;
          double xe[3], jace[9], jite[9];
          map_point_jac(gc, d, n, job.support + (long long)fc.y * pp * d, xie, xe, jace);
          if (!(invert_jac(d, jace, jite) > 0.0))
            atomicExch(bad, 1);
          for (int j = 0; j < d; ++j)
            {
              double s = 0;
              for (int i = 0; i < d; ++i)
                s += normal[i] * jite[i * d + j];
              jne[j] = s;
            }
        }
      for (int j = 0; j < d; ++j)
        {
          if (!job.compress)
            {
              fg[(1 + j) * nqf + q] = job.coefficient ? jni[j] * a : jni[j];
              fg[(1 + d + j) * nqf + q] = job.coefficient ? jne[j] * a : jne[j];
            }
          else if (q == 0)
            {
              fg[1 + j] = jni[j];
              fg[1 + d + j] = jne[j];
            }
        }
    }
  const double p1sq = (double)k * k;
  double tau;
  if (boundary)
    tau = p1sq * area / job.volume[fc.x];
  else
    tau = p1sq * 0.5 * (area / job.volume[fc.x] + area / job.volume[fc.y]);
  if (job.coefficient)
    tau *= abar / (double)nqf;
  job.penalty[f] = tau;
}

// Physical quadrature points of the owned cells, x[c][q][d], and the plain
// det(J) w_q (no coefficient) the forcing integral uses
// (add_forcing, operators.cpp:1115-1145).
__global__ void cell_qpoint_kernel(GeometryJob job, GeoConst gc, double *x_out, double *detw)
{
  const int d = job.d, k = job.k, n = job.m + 1;
  int nq = 1, pp = 1;
  for (int a = 0; a < d; ++a)
    {
      nq *= k;
      pp *= n;
    }
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)job.n_geo_cells * nq)
    return;
  const int c = (int)(gid / nq);
  const int q = (int)(gid - (long long)c * nq);
  double xi[3] = {0, 0, 0};
  int idx = q;
  for (int a = 0; a < d; ++a)
    {
      xi[a] = gc.qp[idx % k];
      idx /= k;
    }
  double x[3], jac[9], jit[9];
  map_point_jac(gc, d, n, job.support + (long long)c * pp * d, xi, x, jac);
  const double det = invert_jac(d, jac, jit);
  if (x_out)
    for (int a = 0; a < d; ++a)
      x_out[gid * d + a] = x[a];
  if (detw)
    detw[gid] = det * cell_weight(gc, d, k, q);
}

// Face quadrature points (GeometryCache::face_qpoints, geometry.cpp:415-453):
// mapped from the interior side, x[f][qf][d].
__global__ void face_qpoint_kernel(GeometryJob job, GeoConst gc, double *x_out)
{
  const int d = job.d, k = job.k, n = job.m + 1;
  int nqf = 1, pp = 1;
  for (int a = 0; a < d - 1; ++a)
    nqf *= k;
  for (int a = 0; a < d; ++a)
    pp *= n;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= job.n_faces * nqf)
    return;
  const long long f = gid / nqf;
  const int q = (int)(gid - f * nqf);
  const int4 fc = job.faces[f];
  const int axis = fc.z / 2;
  double xi[3] = {0, 0, 0};
  int idx = q;
  for (int a = 0, t = 0; a < d; ++a)
    {
      if (a == axis)
        continue;
      xi[a] = gc.qp[idx % k];
      idx /= k;
      ++t;
    }
  xi[axis] = fc.z % 2 ? 1.0 : 0.0;
  double xq[3], jac[9];
  map_point_jac(gc, d, n, job.support + (long long)fc.x * pp * d, xi, xq, jac);
  for (int a = 0; a < d; ++a)
    x_out[gid * d + a] = xq[a];
}

GeoConst make_geo_const(int k, int m)
{
  if (k > 16 || m + 1 > 16 || m < 1)
    fail(Code::invalid_argument, "geometry: k or mapping degree out of range");
  GeoConst gc{};
  const Quad1D g = gauss(k);
  for (int i = 0; i < k; ++i)
    {
      gc.qp[i] = g.points[i];
      gc.qw[i] = g.weights[i];
    }
  const Quad1D gl = gauss_lobatto(m + 1);
  for (int i = 0; i <= m; ++i)
    gc.nodes[i] = gl.points[i];
  return gc;
}

} // namespace

void run_qpoints(const GeometryJob &job, double *cell_x, double *cell_detw, double *face_x,
                 cudaStream_t s)
{
  const GeoConst gc = make_geo_const(job.k, job.m);
  long long nq = 1;
  for (int a = 0; a < job.d; ++a)
    nq *= job.k;
  const int bs = 128;
  const long long nc = (long long)job.n_geo_cells * nq;
  if ((cell_x || cell_detw) && nc > 0)
    cell_qpoint_kernel<<<(unsigned)((nc + bs - 1) / bs), bs, 0, s>>>(job, gc, cell_x, cell_detw);
  const long long nf = job.n_faces * (nq / job.k);
  if (face_x && nf > 0)
    face_qpoint_kernel<<<(unsigned)((nf + bs - 1) / bs), bs, 0, s>>>(job, gc, face_x);
  cuda_check(cudaGetLastError(), "quadrature point kernels");
  cuda_check(cudaStreamSynchronize(s), "quadrature point sync");
}

void run_geometry(const GeometryJob &job, cudaStream_t s)
{
  const GeoConst gc = make_geo_const(job.k, job.m);
  DeviceArray<int> bad(1);
  cuda_check(cudaMemsetAsync(bad.get(), 0, sizeof(int), s), "memset");
  long long nq = 1;
  for (int a = 0; a < job.d; ++a)
    nq *= job.k;
  const long long ncell_threads = (long long)job.n_geo_cells * (job.compress ? 1 : nq);
  const int bs = 128;
  if (job.n_slots > 0)
    volume_kernel<<<(job.n_slots + bs - 1) / bs, bs, 0, s>>>(job, gc, bad.get());
  if (ncell_threads > 0)
    cell_geometry_kernel<<<(unsigned)((ncell_threads + bs - 1) / bs), bs, 0, s>>>(job, gc,
                                                                                 bad.get());
  if (job.n_faces > 0)
    face_geometry_kernel<<<(unsigned)((job.n_faces + bs - 1) / bs), bs, 0, s>>>(job, gc,
                                                                               bad.get());
  cuda_check(cudaGetLastError(), "geometry kernels");
  int h = 0;
  cuda_check(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  cuda_check(cudaStreamSynchronize(s), "geometry sync");
  if (h)
    fail(Code::runtime_error, "precompute_geometry: non-positive mapping Jacobian");
}

} // namespace dgx
