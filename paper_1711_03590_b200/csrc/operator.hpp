// The rank operator: host setup products plus the device state of one
// B200 SIPG-Laplacian apply (the C ABI's dgx_op).
#pragma once

#include "device.hpp"
#include "setup.hpp"

#include "../../include/dgx.h"

#include <memory>
#include <vector>

namespace dgx
{

class Operator
{
public:
  Operator(const dgx_setup &s, int device);
  ~Operator();
  Operator(const Operator &) = delete;
  Operator &operator=(const Operator &) = delete;

  void apply(void *u, void *y, const dgx_hooks *hooks, cudaStream_t stream, bool fp32);
  // phase 1: inner tasks; phase 2: ghost-coupled + ghost-side tasks
  void apply_phase(int phase, const void *u, void *y, cudaStream_t stream, bool fp32);
  void check_apply_args(const void *u, const void *y, bool fp32) const;
  void accumulate_plan(int idx, const double *contrib, double *y, cudaStream_t s);
  // y = A u with host buffers (dgx_apply_host): single-rank 3D layouts run a
  // z-slab pipeline (H2D of slab k+1, apply of slab k, D2H of slab k-1 on
  // three streams); other layouts H2D, both phases, D2H. Blocking.
  void apply_host(const double *u, double *y);

  const RankLayout &layout() const { return layout_; }
  int d() const { return d_; }
  int k() const { return k_; }
  int precision() const { return precision_; }
  int basis() const { return basis_; }
  int kind() const { return kind_; }
  // advection: velocity per quadrature point (device [cell][q][d], [face][qf][d])
  void set_velocity(const double *c_cells, const double *c_faces, cudaStream_t s);
  int device() const { return device_; }
  int n_ranks() const { return n_ranks_; }
  long long nq() const { return nq_; }
  bool compressed() const { return compressed_; }
  bool cartesian_records() const { return cart_; }
  bool host_only() const { return host_only_; }
  // task lists as built on the host: slot, geometry record, 2d face entries
  const std::vector<int> &host_task_slot() const { return host_task_slot_; }
  const std::vector<int> &host_task_geo() const { return host_task_geo_; }
  const std::vector<int2> &host_task_face() const { return host_task_face_; }
  int n_inner() const { return n_inner_; }

  std::vector<double> geometry(int which) const;
  // physical quadrature points: 0 owned cells [cell][q][d], 1 computed faces
  // [face][qf][d], 2 boundary flag per computed face (needs a mapping)
  std::vector<double> quadrature_points(int which);
  // RankOperator::assemble_rhs (operators.cpp:266-282); f: [owned cell][q],
  // g: [computed face][qf] device arrays (null: zero)
  void assemble_rhs(const double *f, const double *g, double *rhs, cudaStream_t s);
  dgx_stats stats() const;

  // exchange plans flattened for the transports: value indices into the
  // rank-local vector (slot * k^d + dof) in plan order, per-plan offsets in
  // values (size plans + 1)
  const DeviceArray<long long> &send_index() const { return send_index_; }
  const DeviceArray<long long> &recv_index() const { return recv_index_; }
  const std::vector<long long> &send_offsets() const { return send_offsets_; }
  const std::vector<long long> &recv_offsets() const { return recv_offsets_; }
  // whole ghost cells arrive in ghost storage order: receive in place
  bool recv_in_place() const { return recv_in_place_; }
  // whole-cell plans: send cells as slot lists, per-plan offsets in cells
  bool whole_cells() const { return layout_.whole_cells; }
  const DeviceArray<int> &send_slots() const { return send_slots_; }
  const std::vector<long long> &send_cell_offsets() const { return send_cell_offsets_; }
  // the ghost-coupled phase of an exchanged apply runs on this stream
  // (highest priority, created on first use), concurrent with phase 1
  cudaStream_t ghost_stream();

private:
  void build_tasks(const std::vector<RawFace> &faces, const Partition &part);
  void build_geometry(const dgx_setup &s, const std::vector<RawFace> &faces);
  template <typename Real>
  void launch_range(int begin, int count, const Real *u, Real *y, cudaStream_t s);
  template <typename Real>
  void launch_tasks(const int *slot, const int *geo, const int2 *face, int count, const Real *u,
                    Real *y, cudaStream_t s);

  // host-buffer pipeline state (apply_host), built on first use
  struct HostPipe
  {
    bool built = false, pipelined = false, periodic_z = false;
    int nchunk = 0;
    std::vector<int> task_begin;       // per chunk, into the chunk-ordered task arrays (+ end)
    std::vector<long long> cell_begin; // per chunk, first owned cell (+ end)
    DeviceArray<int> slot, geo;
    DeviceArray<int2> face;
    DeviceArray<double> du, dy;
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    std::vector<cudaEvent_t> ev_h, ev_c;
  } pipe_;
  void build_host_pipe();

  MeshDesc mesh_;
  int d_ = 3, p_ = 1, k_ = 2, precision_ = 0, device_ = 0, n_ranks_ = 1, basis_ = 0;
  int kind_ = 0; // 0 Laplacian, 1 advection
  bool sym_ = false; // geometry variant g4 (merged symmetric coefficient)
  double velocity_[3] = {1, 1, 1};
  bool variable_velocity_ = false;
  DeviceArray<double> normals_;           // advection: [face][d][qf or 1]
  DeviceArray<double> adv_cell_, adv_face_; // advection records
  long long nq_ = 0, nqf_ = 0;
  RankLayout layout_;
  bool compressed_ = false;
  bool cart_ = false; // compressed records axis-aligned (CART kernels)
  bool tensor_ = false; // ... run the tensor-product kernel (sipg_cart.cuh)
  bool host_only_ = false;
  std::vector<int> host_task_slot_, host_task_geo_;
  std::vector<int2> host_task_face_;

  DeviceArray<double> cell_geo_, face_geo_, penalty_;
  DeviceArray<float> cell_geo_f_, face_geo_f_, penalty_f_;
  DeviceArray<int> task_slot_, task_geo_;
  DeviceArray<int2> task_face_;
  int n_inner_ = 0, n_coupled_ = 0;

  // mapping kept for quadrature points / right-hand side (not for
  // HOST_ARRAYS geometry)
  bool has_mapping_ = false;
  int map_degree_ = 1;
  DeviceArray<double> support_;
  DeviceArray<int4> face_list_;
  DeviceArray<double> cell_detw_; // det(J) w_q per owned cell point, lazily
  std::vector<char> face_boundary_;
  void ensure_detw();
  GeometryJob mapping_job() const;

  DeviceArray<long long> send_index_, recv_index_;
  std::vector<long long> send_offsets_, recv_offsets_; // in values, size plans+1
  bool recv_in_place_ = true;
  DeviceArray<int> send_slots_;
  std::vector<long long> send_cell_offsets_;
  cudaStream_t ghost_stream_ = nullptr;
};

// solvers.cu
dgx_solve_report conjugate_gradient(Operator &op, const double *b, double *x, double rel_tol,
                                    int max_iterations, cudaStream_t s);

} // namespace dgx
