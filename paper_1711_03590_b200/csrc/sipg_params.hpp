// Parameters of the fused SIPG apply kernel (shared by the host side).
#pragma once

#include <cuda_runtime.h>

namespace dgx
{
namespace dev
{

// ---- kernel parameters ---------------------------------------------------

// task_face[t * 2D + phi]: x = neighbour slot, or -1 (boundary face), or -2
// (face not computed on this rank: its contribution arrives by compress);
// y = local face record | (own side << 30).
template <typename Real>
struct ApplyParams
{
  const Real *u;
  Real *y;
  const Real *cell_geo; // [geo][D*D+1][NQ] or compressed [geo][D*D+1]
  const Real *face_geo; // [face][2D+1][P]: JxW_f, n.J^{-T}(e-), n.J^{-T}(e+)
  const Real *penalty;  // [face]
  const int *task_slot;
  const int *task_geo;  // cell geometry record, -1: no cell integral
  const int2 *task_face;
  int n_tasks;
  int n_owned; // slots >= n_owned are ghost cells (ghost-side tasks)
  int sym;     // 1: cell records hold the g4 coefficient [geo][d(d+1)/2][NQ]
  int ahead;   // tasks resident on the device at once (set by the launcher)
  int cart;    // 1: axis-aligned affine records (Operator::cart_), CART kernels
};

// Advection apply (OperatorKind::advection, operators.cpp:634-667 cell,
// :942-960 interior faces, :1033-1060 boundary faces).
template <typename Real>
struct AdvParams
{
  const Real *u;
  Real *y;
  const Real *cell; // [geo][D][NQ] or compressed [geo][D]: J^{-1} c det(J) w (no w if compressed)
  const Real *face; // [face][2][P] or compressed [face][2]: JxW_f (no w if compressed), c.n
  const int *task_slot;
  const int *task_geo;
  const int2 *task_face;
  int n_tasks;
  int n_owned;
};

// Right-hand side assembly (assemble_rhs, operators.cpp:266-282): forcing
// f at the owned cells' quadrature points times det(J) w_q, Dirichlet data g
// at the computed faces' quadrature points (boundary faces only).
template <typename Real>
struct RhsParams
{
  const Real *f;    // [slot][q] or null
  const Real *detw; // [slot][q]
  const Real *g;    // [local face][qf] or null
  Real *y;
  const Real *face_geo; // Laplacian face records, or the advection ones (AdvParams::face)
  const Real *penalty;
  const int *task_slot;
  const int2 *task_face;
  int n_tasks;
};

} // namespace dev
} // namespace dgx
