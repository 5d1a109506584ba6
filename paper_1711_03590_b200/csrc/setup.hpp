// Host-side setup of the B200 SIPG-Laplacian operator: 1D numerics, mesh
// topology, partition, ghost layout and exchange plans. Everything here is
// computed once per operator; the apply itself runs on the device.
//
// The topology routines reproduce the reference bit for bit (face order,
// slabs, face owners, ghost order, plan order) because the ghost maps and
// DoF indexing must be identical (BASELINE.json north star).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace dgx
{

enum class Code
{
  ok = 0,
  invalid_argument = 1, // std::invalid_argument in the reference
  logic_error = 2,      // std::logic_error
  runtime_error = 3,    // std::runtime_error
  cuda_error = 4
};

struct Error : std::runtime_error
{
  Code code;
  Error(Code c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(Code c, const std::string &m) { throw Error(c, m); }

inline constexpr std::uint32_t invalid_cell = 0xffffffffu;

// ---------------------------------------------------------------- 1D ----

struct Quad1D
{
  std::vector<double> points, weights;
};

// Gauss-Legendre / Gauss-Lobatto on [0,1], Newton on Legendre polynomials
// followed by exact symmetrization (reference quadrature.cpp:56-127).
Quad1D gauss(int n);
Quad1D gauss_lobatto(int n);

// Tables of the nodal Gauss-Lobatto basis of degree p on k = p+1 Gauss
// points (basis.cpp:261-325), plus the collocation-space rows the device
// kernels use for face traces.
// basis: 0 lagrange_gauss_lobatto, 1 lagrange_gauss, 2 hermite_like
// (make_basis, basis.cpp:116-180). The Hermite-like functions are stored
// sign-flipped, psi_j = sigma_j phi_j with sigma_{k-2} = -1 (hermite_sign),
// which makes S and D mirror-(skew-)symmetric; the kernel multiplies vector
// entries by the per-dof sign on load and store.
struct Tables1D
{
  int k = 0;
  int basis = 0;
  std::vector<double> S;   // k x k, S[q][j] = phi_j(x_q)
  std::vector<double> Dco; // k x k, collocation derivative in the Gauss points
  std::vector<double> D;   // k x k, D[q][j] = phi_j'(x_q) (nodal derivative)
  std::array<std::vector<double>, 2> Sf, Df; // nodal value / derivative rows at x=0,1
  // rf[s] = Sf[s] S^{-1}: extrapolation of Gauss-point values to the end
  // point s (exact for polynomials of degree < k).
  std::array<std::vector<double>, 2> rf;
  std::vector<double> qw; // Gauss weights
};
Tables1D make_tables(int p, int basis);
int hermite_sign(int k, int j);

// ------------------------------------------------------------ mesh ------

// Mirror of dg::RawFace (mesh.hpp:80-93); identical 12-byte layout.
struct RawFace
{
  std::uint32_t interior_cell = invalid_cell;
  std::uint32_t exterior_cell = invalid_cell;
  std::uint8_t interior_face_number = 0;
  std::uint8_t exterior_face_number = 0;
  std::uint8_t subface_index = 255;
  std::uint8_t face_orientation = 0;
  bool at_boundary() const { return exterior_cell == invalid_cell; }
};
static_assert(sizeof(RawFace) == 12, "RawFace must match the reference layout");

struct MeshDesc
{
  int d = 3;
  std::array<int, 3> cells{1, 1, 1};
  std::array<double, 3> lo{0, 0, 0}, hi{1, 1, 1};
  double amplitude = 0.0; // reference bump a * prod sin(pi y) (mesh.cpp:11-26)
  int mapping_degree = 1;
  std::array<bool, 3> periodic{false, false, false};
  std::array<int, 6> dirichlet_id{0, 1, 2, 3, 4, 5};

  long long n_cells() const
  {
    long long n = 1;
    for (int a = 0; a < d; ++a)
      n *= cells[a];
    return n;
  }
  void check() const;
};

// enumerate_faces (mesh.cpp:70-132): axis by axis, cells lexicographic.
std::vector<RawFace> enumerate_faces(const MeshDesc &m);

struct Partition
{
  int n_ranks = 1;
  std::vector<int> cell_owner;
  std::vector<std::pair<int, int>> ranges;
  std::vector<int> face_owner;
};
// partition_cells + assign_face_owners (mesh.cpp:134-232).
Partition make_partition(const MeshDesc &m, const std::vector<RawFace> &faces,
                         int n_ranks);
void assign_face_owners(const std::vector<RawFace> &faces, Partition &p);

// ------------------------------------------------- layout and plans -----

// ExchangePlan::NeighborPlan (ghost_exchange.hpp:29-52): cells ascending,
// dof_offsets[i]..dof_offsets[i+1] the cell-local dofs of cells[i] that
// travel (whole cells for the nodal / generic bases with a face normal
// derivative, two layers per coupled face for the Hermite-like basis,
// ghost_exchange.cpp:49-144).
struct NeighborPlan
{
  int neighbor = -1;
  std::vector<std::uint32_t> cells;
  std::vector<std::uint32_t> dof_offsets;
  std::vector<std::uint32_t> dofs;
  long long n_values() const { return (long long)dofs.size(); }
};

// Rank-local layout with the reference W=1 numbering (dof_layout.cpp:50-65,
// 170-253): owned cells cell-major, ghosts appended in ascending global id.
struct RankLayout
{
  int rank = 0;
  long long dofs_per_cell = 0;
  std::uint32_t owned_begin = 0, n_owned = 0;
  std::vector<std::uint32_t> ghosts;     // ascending
  std::vector<int> ghost_owner;
  std::vector<std::uint32_t> my_faces;   // face ids computed on this rank
  std::vector<NeighborPlan> send, recv;  // ascending neighbour rank
  bool whole_cells = true;               // every plan ships complete cells

  long long owned_size() const { return (long long)n_owned * dofs_per_cell; }
  long long total_size() const
  {
    return owned_size() + (long long)ghosts.size() * dofs_per_cell;
  }
  // local slot of a global cell (owned first, then ghosts); -1 if absent
  long long slot(std::uint32_t global) const;
};

// kind: 0 Laplacian (values and first derivatives), 1 advection (values):
// ghost_need, ghost_exchange.cpp:13-24
RankLayout build_layout(const MeshDesc &m, const std::vector<RawFace> &faces,
                        const Partition &p, int rank, int k, int basis, int kind = 0);

// Mapping support points [cell][(m+1)^d][d] on Gauss-Lobatto nodes of
// degree m for the listed global cells (build_mapping, geometry.cpp:36-63,
// with Mesh::map_point, mesh.cpp:11-26).
std::vector<double> reference_support(const MeshDesc &m,
                                      const std::vector<std::uint32_t> &cells);
// BASELINE.json vertex deformation x + eps h prod sin(2 pi x_a) (m = 1).
std::vector<double> vertex_bump_support(const MeshDesc &m, double eps,
                                        const std::vector<std::uint32_t> &cells);

} // namespace dgx
