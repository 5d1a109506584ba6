// Device-side helpers shared by the operator implementation.
#pragma once

#include "setup.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace dgx
{

inline void cuda_check(cudaError_t e, const char *what)
{
  if (e != cudaSuccess)
    fail(Code::cuda_error, std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device allocation (no torch types cross the C ABI; the operator
// owns geometry and task tables, the caller owns the vectors).
template <typename T>
class DeviceArray
{
public:
  DeviceArray() = default;
  explicit DeviceArray(size_t n) { resize(n); }
  DeviceArray(const DeviceArray &) = delete;
  DeviceArray &operator=(const DeviceArray &) = delete;
  DeviceArray(DeviceArray &&o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceArray &operator=(DeviceArray &&o) noexcept
  {
    if (this != &o)
      {
        release();
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
      }
    return *this;
  }
  ~DeviceArray() { release(); }

  void resize(size_t n)
  {
    release();
    if (n)
      cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
    n_ = n;
  }
  void upload(const T *h, size_t n, cudaStream_t s = nullptr)
  {
    if (n != n_)
      resize(n);
    if (n)
      cuda_check(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s),
                 "upload");
  }
  void upload(const std::vector<T> &v, cudaStream_t s = nullptr) { upload(v.data(), v.size(), s); }
  std::vector<T> download() const
  {
    std::vector<T> h(n_);
    if (n_)
      cuda_check(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "download");
    return h;
  }
  T *get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

private:
  void release()
  {
    if (p_)
      cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T *p_ = nullptr;
  size_t n_ = 0;
};

namespace dev
{
template <typename Real>
struct ApplyParams;
template <typename Real>
struct RhsParams;
template <typename Real>
struct AdvParams;
}

// sipg.cu (kernels in sipg_gl.cu / sipg_gauss.cu / sipg_hermite.cu);
// basis: 0 lagrange_gauss_lobatto, 1 lagrange_gauss, 2 hermite_like
void upload_tables(int K, int basis);
int kernel_cells_per_cta(int D, int K, bool cart = false);
// brick size of the pencil-pair kernel's CTAs (0: none; 4: 2x2x1; 8: 2x2x2)
int kernel_brick(int D, int K);
template <typename Real>
void launch_apply(int D, int K, int basis, bool compressed, const dev::ApplyParams<Real> &prm,
                  cudaStream_t s);
void launch_rhs(int D, int K, int basis, bool compressed, bool adv,
                const dev::RhsParams<double> &prm, cudaStream_t s);
void launch_adv(int D, int K, int basis, bool compressed, const dev::AdvParams<double> &prm,
                cudaStream_t s);
// advection.cu: cell coefficient J^{-1} c det(J) w [geo][d][q] (or [geo][d]
// compressed) and face records (JxW_f, c.n) [face][2][qf] (or [face][2]) from
// the g3 arrays, the unit normals and the velocity (constant, or per point)
void run_adv_coefficients(int d, int k, bool compressed, long long n_cells, long long n_faces,
                          const double *cell_geo, const double *face_geo,
                          const double *normals, const double velocity[3],
                          const double *c_cells, const double *c_faces, double *adv_cell,
                          double *adv_face, cudaStream_t s);

// geometry.cu -- device precompute of the g3 arrays from mapping support
// points (reference geometry.cpp:36-150,248-522), written straight into the
// device SoA layout the apply kernel reads.
struct GeometryJob
{
  int d = 3, k = 2, m = 1;
  bool compress = false;
  int coefficient = 0;  // 1: a(x) = 1 + 0.5 sin(pi x) cos(pi y) folded in
  bool g4 = false;      // cell records: merged symmetric coefficient (variant g4)
  double cart_volume = 0; // > 0: Cartesian mesh, every cell has this volume
  const double *support = nullptr; // device [n_slots][(m+1)^d][d]
  int n_slots = 0;       // local cells with support points
  int n_geo_cells = 0;   // owned cells, slots 0..n_geo_cells-1
  long long n_faces = 0; // faces computed on this rank
  const int4 *faces = nullptr; // device: (slot-, slot+ or -1, fn-, fn+)
  double *cell_geo = nullptr;  // [n_geo][d*d+1][k^d] or [n_geo][d*d+1]
  double *face_geo = nullptr;  // [n_faces][2d+1][k^{d-1}]
  double *penalty = nullptr;   // [n_faces]
  double *volume = nullptr;    // scratch [n_slots]
  double *face_normal = nullptr; // optional [n_faces][d][k^{d-1} or 1] unit normals (e-)
};
void run_geometry(const GeometryJob &job, cudaStream_t s);
// physical quadrature points of the owned cells ([cell][q][d]) with the
// plain det(J) w_q ([cell][q]), and of the computed faces ([face][qf][d]);
// any output may be null
void run_qpoints(const GeometryJob &job, double *cell_x, double *cell_detw, double *face_x,
                 cudaStream_t s);

// exchange.cu -- halo pack / unpack / compress kernels over the flat value
// index lists of the exchange plans (slot * k^d + cell-local dof, in plan
// order: ascending cells, ascending dofs, ghost_exchange.cpp:240-295).
template <typename T>
void launch_gather_values(const T *src, const long long *index, long long n, T *dst,
                          cudaStream_t s);
template <typename T>
void launch_scatter_values(T *dst, const long long *index, long long n, const T *src,
                           cudaStream_t s);
template <typename T>
void launch_scatter_add_values(T *dst, const long long *index, long long n, const T *src,
                               cudaStream_t s);
// whole-cell plans: cell slot lists (value i = dof i % nq of cell i / nq)
template <typename T>
void launch_gather_cells(const T *src, const int *slot, long long n_cells, int nq, T *dst,
                         cudaStream_t s);
template <typename T>
void launch_scatter_add_cells(T *dst, const int *slot, long long n_cells, int nq, const T *src,
                              cudaStream_t s);
template <typename Real>
void launch_convert(const double *src, Real *dst, long long n, cudaStream_t s);
// compressed g3 records that are not axis-aligned (0: Operator::cart_)
long long count_non_axis_records(int d, const double *cell_geo, long long n_cells, const double *face_geo,
                                 const signed char *face_axis, long long n_faces);

} // namespace dgx
