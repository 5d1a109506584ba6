// Setup of the advection operator's device records (OperatorKind::advection,
// reference operators.cpp:397-545, 634-667): the cell coefficient
// J^{-1} c det(J) w per quadrature point -- the g3 algebra of cell_advection
// folded once (the reference's g4 coefficient, geometry.cpp:370-388) -- and
// per face point (JxW_f, c.n) with the unit normal of the interior side
// (load_face_geometry, operators.cpp:502-543).
#include "device.hpp"

namespace dgx
{
namespace
{
__global__ void adv_cell_kernel(int d, long long nrec, long long n_cells, const double *cell_geo,
                                double c0, double c1, double c2, const double *c_cells,
                                double *adv)
{
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= n_cells * nrec)
    return;
  const long long c = gid / nrec, r = gid - c * nrec;
  const int nc = d * d + 1;
  const double *g = cell_geo + c * nc * nrec + r;
  double v[3] = {c0, c1, c2};
  if (c_cells)
    for (int a = 0; a < d; ++a)
      v[a] = c_cells[gid * d + a];
  const double jxw = g[d * d * nrec];
  for (int i = 0; i < d; ++i)
    {
      // (J^{-T})^T c = J^{-1} c (advection_cell_integrand, geometry.cpp:175-186)
      double acc = g[i * nrec] * v[0];
      for (int j = 1; j < d; ++j)
        acc += g[(j * d + i) * nrec] * v[j];
      adv[(c * d + i) * nrec + r] = acc * jxw;
    }
}

__global__ void adv_face_kernel(int d, long long nrf, long long n_faces, const double *face_geo,
                                const double *normals, double c0, double c1, double c2,
                                const double *c_faces, double *adv)
{
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= n_faces * nrf)
    return;
  const long long f = gid / nrf, q = gid - f * nrf;
  double v[3] = {c0, c1, c2};
  if (c_faces)
    for (int a = 0; a < d; ++a)
      v[a] = c_faces[gid * d + a];
  double s = 0;
  for (int i = 0; i < d; ++i)
    s += v[i] * normals[(f * d + i) * nrf + q];
  adv[(f * 2) * nrf + q] = face_geo[f * (2 * d + 1) * nrf + q];
  adv[(f * 2 + 1) * nrf + q] = s;
}
} // namespace

void run_adv_coefficients(int d, int k, bool compressed, long long n_cells, long long n_faces,
                          const double *cell_geo, const double *face_geo,
                          const double *normals, const double velocity[3],
                          const double *c_cells, const double *c_faces, double *adv_cell,
                          double *adv_face, cudaStream_t s)
{
  long long nq = 1;
  for (int a = 0; a < d; ++a)
    nq *= k;
  const long long nrec = compressed ? 1 : nq, nrf = compressed ? 1 : nq / k;
  const int bs = 128;
  if (n_cells > 0)
    adv_cell_kernel<<<(unsigned)((n_cells * nrec + bs - 1) / bs), bs, 0, s>>>(
      d, nrec, n_cells, cell_geo, velocity[0], velocity[1], velocity[2], c_cells, adv_cell);
  if (n_faces > 0)
    adv_face_kernel<<<(unsigned)((n_faces * nrf + bs - 1) / bs), bs, 0, s>>>(
      d, nrf, n_faces, face_geo, normals, velocity[0], velocity[1], velocity[2], c_faces,
      adv_face);
  cuda_check(cudaGetLastError(), "advection coefficient kernels");
  cuda_check(cudaStreamSynchronize(s), "advection coefficients");
}

} // namespace dgx
