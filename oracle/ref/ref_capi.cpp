// Test-infrastructure C ABI over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/ref/Makefile
// into oracle/_ref/libdgref.so). Only tests/, tests/golden/make_golden.py,
// __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs load
// this library; the product (paper_1711_03590_b200/) never does.
//
// Every entry point returns 0 on success and -1 on a C++ exception, whose
// message is available from dgref_last_error().
//
// The "world" mirrors the reference's own test fixtures:
//   * SingleRankOp / SerialRanks  (proj/tests/test_operators.cpp:26-39,446-535)
//   * DistWorld + distributed_apply (proj/tests/test_ghost_exchange.cpp:20-87)
//   * BenchWorld::run              (proj/src/bench.cpp:104-166)
// with the nodal Gauss-Lobatto basis forced unless
// dgref_set_basis selected another BasisKind (or -1: the reference default
// of make_operator_config, Hermite-like for the Laplacian at p >= 3,
// operators.cpp:27-41) for the worlds created after it.

#include <dg/basis.hpp>
#include <dg/geometry.hpp>
#include <dg/ghost_exchange.hpp>
#include <dg/mesh.hpp>
#include <dg/operators.hpp>
#include <dg/oracle.hpp>
#include <dg/quadrature.hpp>
#include <dg/solvers.hpp>

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

using namespace dg;

namespace
{
thread_local std::string g_err;
thread_local int g_basis = 0; // BasisKind for new worlds; -1 = reference default
thread_local int g_manufactured = 0; // forcing/dirichlet of the convergence study
thread_local int g_kind = 0;          // 0 laplacian, 1 advection
thread_local int g_variant = 3;       // geometry variant of new worlds: 3 g3, 4 g4
thread_local double g_velocity[3] = {1, 1, 1};
thread_local int g_velocity_field = 0; // 1: the variable test field below

// Variable transport field used by the advection tests (test input).
std::array<double, 3> test_velocity(const std::array<double, 3> &x)
{
  return {1.0 + 0.3 * std::sin(2.0 * M_PI * x[1]), 0.7 + 0.2 * std::cos(2.0 * M_PI * x[0]),
          0.4 + 0.1 * x[0] * x[1]};
}

// The manufactured solution of the reference convergence study
// (bench.cpp:437-459), restated here as test input.
double mf_solution(int d, const std::array<double, 3> &x)
{
  double u = std::cos(2.3 * x[0] + 0.4);
  u *= std::cos(1.7 * x[1] - 0.2);
  if (d == 3)
    u *= std::cos(1.1 * x[2] + 0.1);
  return u;
}
std::array<double, 3> mf_gradient(int d, const std::array<double, 3> &x)
{
  const double c0 = std::cos(2.3 * x[0] + 0.4), s0 = std::sin(2.3 * x[0] + 0.4);
  const double c1 = std::cos(1.7 * x[1] - 0.2), s1 = std::sin(1.7 * x[1] - 0.2);
  const double c2 = d == 3 ? std::cos(1.1 * x[2] + 0.1) : 1.0;
  const double s2 = d == 3 ? std::sin(1.1 * x[2] + 0.1) : 0.0;
  return {-2.3 * s0 * c1 * c2, -1.7 * c0 * s1 * c2, d == 3 ? -1.1 * c0 * c1 * s2 : 0.0};
}
double mf_neg_laplacian(int d, const std::array<double, 3> &x)
{
  const double lam = 2.3 * 2.3 + 1.7 * 1.7 + (d == 3 ? 1.1 * 1.1 : 0.0);
  return lam * mf_solution(d, x);
}

template <typename F>
int guard(F &&f)
{
  try
    {
      f();
      return 0;
    }
  catch (const std::exception &e)
    {
      g_err = e.what();
      return -1;
    }
  catch (...)
    {
      g_err = "unknown exception";
      return -1;
    }
}

struct World
{
  Mesh mesh;
  OperatorConfig cfg;
  std::vector<RawFace> faces;
  Partition partition;
  std::shared_ptr<const GeometryCache> geom;
  std::vector<std::unique_ptr<RankOperator>> ops;
  std::vector<ExchangePlan> plans;
  std::vector<DoFLayout> layouts; // topology-only worlds (no operators)
  bool external_geometry = false;
};

const DoFLayout &layout_of(const World &w, int rank)
{
  if (!w.layouts.empty())
    return w.layouts.at(rank);
  return w.ops.at(rank)->layout();
}

long long ipow(int b, int e)
{
  long long r = 1;
  while (e--)
    r *= b;
  return r;
}

void finish_world(World &w, int n_ranks)
{
  for (int r = 0; r < n_ranks; ++r)
    w.ops.push_back(std::make_unique<RankOperator>(w.mesh, w.partition,
                                                   w.faces, w.geom, w.cfg, r));
  const FaceAccess access = make_basis(w.cfg.basis, w.cfg.p).face_access;
  for (int r = 0; r < n_ranks; ++r)
    w.plans.push_back(build_exchange_plan(w.ops[r]->layout(), w.faces,
                                          w.partition, access,
                                          ghost_need(w.cfg.kind)));
}

World *make_world_common(int d, const int *cells, double amplitude,
                         int mapping_degree, int periodic, int p, int n_ranks,
                         int W)
{
  auto w = std::make_unique<World>();
  std::array<BoundarySpec, 6> boundary{};
  for (int s = 0; s < 6; ++s)
    {
      boundary[s].periodic = periodic != 0;
      boundary[s].dirichlet_id = s;
    }
  w->mesh = build_mesh(d, {cells[0], cells[1], d > 2 ? cells[2] : 1},
                       {0, 0, 0}, {1, 1, 1}, amplitude, mapping_degree,
                       boundary);
  const OperatorKind kind = g_kind == 1 ? OperatorKind::advection : OperatorKind::laplacian;
  w->cfg = make_operator_config(kind, d, p, W,
                                g_variant == 4 ? GeometryVariant::g4 : GeometryVariant::g3);
  if (g_basis >= 0)
    w->cfg.basis = static_cast<BasisKind>(g_basis); // GL unless selected
  if (kind == OperatorKind::advection)
    {
      w->cfg.velocity.constant = {g_velocity[0], g_velocity[1], g_velocity[2]};
      if (g_velocity_field == 1)
        w->cfg.velocity.field = test_velocity;
    }
  if (g_manufactured)
    {
      w->cfg.dirichlet = [d](const std::array<double, 3> &x) { return mf_solution(d, x); };
      if (kind == OperatorKind::laplacian)
        w->cfg.forcing = [d](const std::array<double, 3> &x) { return mf_neg_laplacian(d, x); };
      else
        {
          const VelocityField vel = w->cfg.velocity;
          w->cfg.forcing = [d, vel](const std::array<double, 3> &x) {
            const std::array<double, 3> g = mf_gradient(d, x), c = vel(x);
            double f = 0;
            for (int a = 0; a < d; ++a)
              f += c[a] * g[a];
            return f;
          };
        }
    }
  w->faces = enumerate_faces(w->mesh);
  w->partition = partition_cells(w->mesh, n_ranks);
  assign_face_owners(w->mesh, w->faces, w->partition);
  return w.release();
}

} // namespace

extern "C" {

const char *dgref_last_error() { return g_err.c_str(); }

// std::mt19937(seed) + uniform_real_distribution<double>(-1,1), the
// reference's input convention (proj/tests/test_helpers.hpp:11-19).
int dgref_random_vector(long long n, unsigned seed, double *out)
{
  return guard([&] {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (long long i = 0; i < n; ++i)
      out[i] = dist(rng);
  });
}

int dgref_gauss(int n, int lobatto, double *points, double *weights)
{
  return guard([&] {
    const Quadrature1D q =
      lobatto ? gauss_lobatto_quadrature(n) : gauss_quadrature(n);
    std::memcpy(points, q.points.data(), sizeof(double) * n);
    std::memcpy(weights, q.weights.data(), sizeof(double) * n);
  });
}

// Basis of the worlds created next: 0 lagrange_gauss_lobatto (default),
// 1 lagrange_gauss, 2 hermite_like, -1 make_operator_config's choice.
int dgref_set_basis(int kind)
{
  return guard([&] {
    if (kind < -1 || kind > 2)
      throw std::invalid_argument("dgref_set_basis: unknown basis kind");
    g_basis = kind;
  });
}

// Operator of the worlds created next: kind 0 Laplacian, 1 advection with the
// constant velocity c (field 1: the variable test field above).
int dgref_set_operator(int kind, const double *c, int field)
{
  return guard([&] {
    if (kind != 0 && kind != 1)
      throw std::invalid_argument("dgref_set_operator: unknown kind");
    g_kind = kind;
    if (c)
      for (int a = 0; a < 3; ++a)
        g_velocity[a] = c[a];
    g_velocity_field = field;
  });
}

// Geometry variant of the worlds created next (3: g3, 4: g4; the reference's
// precompute_geometry stores the merged coefficient for g4,
// geometry.cpp:370-388).
int dgref_set_variant(int variant)
{
  return guard([&] {
    if (variant != 3 && variant != 4)
      throw std::invalid_argument("dgref_set_variant: g3 or g4");
    g_variant = variant;
  });
}

// Worlds created next carry the manufactured forcing / Dirichlet data of the
// convergence study (bench.cpp:525-560) when flag != 0.
int dgref_set_manufactured(int flag)
{
  return guard([&] { g_manufactured = flag; });
}

// Shape matrices of the selected basis (dgref_set_basis; -1 resolves as for
// the Laplacian) on k-point Gauss quadrature (basis.cpp:261-325):
// S, D (k x k), Dco (k x k), Sf[0..1], Df[0..1] (k each), row-major.
int dgref_shape_matrices(int p, double *S, double *D, double *Dco,
                         double *Sf, double *Df)
{
  return guard([&] {
    const BasisKind kind = g_basis >= 0 ? static_cast<BasisKind>(g_basis)
                           : p >= 3     ? BasisKind::hermite_like
                                        : BasisKind::lagrange_gauss_lobatto;
    const Basis1D b = make_basis(kind, p);
    const ShapeMatrices1D sm = shape_matrices(b, gauss_quadrature(p + 1));
    const int k = p + 1;
    std::memcpy(S, sm.S.data(), sizeof(double) * k * k);
    std::memcpy(D, sm.D.data(), sizeof(double) * k * k);
    std::memcpy(Dco, sm.Dco.data(), sizeof(double) * k * k);
    for (int f = 0; f < 2; ++f)
      {
        std::memcpy(Sf + f * k, sm.Sf[f].data(), sizeof(double) * k);
        std::memcpy(Df + f * k, sm.Df[f].data(), sizeof(double) * k);
      }
  });
}

// World on a reference box mesh with the reference's own geometry
// (precompute_geometry, variant g3, Laplacian).
int dgref_world_create(int d, const int *cells, double amplitude,
                       int mapping_degree, int periodic, int p, int n_ranks,
                       int W, void **out)
{
  return guard([&] {
    std::unique_ptr<World> w(make_world_common(d, cells, amplitude,
                                               mapping_degree, periodic, p,
                                               n_ranks, W));
    w->geom = std::make_shared<GeometryCache>(precompute_geometry(
      w->mesh, w->faces, w->cfg.k(), w->cfg.k(), w->cfg.geometry,
      w->cfg.equation(), w->cfg.velocity));
    finish_world(*w, n_ranks);
    *out = w.release();
  });
}

// World whose g3 geometry arrays are injected (RankOperator accepts any
// GeometryCache matching k, l, equation and variant, operators.cpp:102-105).
// Used for the BASELINE vertex deformation and the folded a(x) coefficient,
// which the reference mesh cannot express.
// compressed: 1 record per cell with jxw = det only (geometry.cpp:267-275).
int dgref_world_create_ext(int d, const int *cells, int periodic, int p,
                           int n_ranks, int W, int compressed,
                           const double *inv_jac_t, const double *jxw,
                           const double *face_jxw, const double *face_jni,
                           const double *face_jne, const double *penalty,
                           void **out)
{
  return guard([&] {
    std::unique_ptr<World> w(
      make_world_common(d, cells, 0.0, 1, periodic, p, n_ranks, W));
    auto g = std::make_shared<GeometryCache>();
    const int k = p + 1;
    g->d = d;
    g->k = k;
    g->l = k;
    g->equation = Equation::laplacian;
    g->variant = w->cfg.geometry; // g3, or g4 (dgref_set_variant)
    g->compression = compressed ? GeometryCompression::cartesian
                                : GeometryCompression::general;
    g->quad1d = gauss_quadrature(k);
    g->n_cells = w->mesh.n_cells();
    g->n_faces = static_cast<long long>(w->faces.size());
    g->n_q_face = ipow(k, d - 1);
    const long long nq = ipow(k, d);
    g->n_q_cell = compressed ? 1 : nq;
    g->wq_cell.resize(nq);
    for (long long q = 0; q < nq; ++q)
      {
        double wgt = 1.0;
        long long idx = q;
        for (int a = 0; a < d; ++a)
          {
            wgt *= g->quad1d.weights[idx % k];
            idx /= k;
          }
        g->wq_cell[q] = wgt;
      }
    g->wq_face.resize(g->n_q_face);
    for (long long q = 0; q < g->n_q_face; ++q)
      {
        double wgt = 1.0;
        long long idx = q;
        for (int a = 0; a < d - 1; ++a)
          {
            wgt *= g->quad1d.weights[idx % k];
            idx /= k;
          }
        g->wq_face[q] = wgt;
      }
    const long long nrec = static_cast<long long>(g->n_cells) * g->n_q_cell;
    g->inv_jac_t.assign(inv_jac_t, inv_jac_t + nrec * d * d);
    g->jxw.assign(jxw, jxw + nrec);
    if (g->variant == GeometryVariant::g4)
      {
        // the merged coefficient of the injected g3 data, formed exactly as
        // precompute_geometry does (symmetric_coefficient, geometry.cpp:219-246)
        const int ns = n_symmetric_entries(d);
        const int ii[6] = {0, 1, 2, 0, 0, 1}, jj[6] = {0, 1, 2, 1, 2, 2};
        const int ii2[3] = {0, 1, 0}, jj2[3] = {0, 1, 1};
        g->coeff.resize(nrec * ns);
        for (long long r = 0; r < nrec; ++r)
          for (int e = 0; e < ns; ++e)
            {
              const int i = d == 3 ? ii[e] : ii2[e], j = d == 3 ? jj[e] : jj2[e];
              double s = 0;
              for (int a = 0; a < d; ++a)
                s += inv_jac_t[r * d * d + a * d + i] * inv_jac_t[r * d * d + a * d + j];
              g->coeff[r * ns + e] = s * jxw[r];
            }
      }
    const long long nf = g->n_faces * g->n_q_face;
    g->face_jxw.assign(face_jxw, face_jxw + nf);
    g->face_jni.assign(face_jni, face_jni + nf * d);
    g->face_jne.assign(face_jne, face_jne + nf * d);
    g->penalty.assign(penalty, penalty + g->n_faces);
    w->geom = g;
    w->external_geometry = true;
    finish_world(*w, n_ranks);
    *out = w.release();
  });
}

// Topology only (no geometry, no operator): mesh, faces, partition, face
// owners, every rank's DoFLayout (build_dof_layout, W = 1) and exchange
// plans (build_exchange_plan) -- the bit-exact maps at sizes where the
// geometry precompute would take an hour (dof_layout.cpp:170-253,
// ghost_exchange.cpp:100-144, mesh.cpp:70-232).
int dgref_topology_create(int d, const int *cells, int periodic, int p, int n_ranks, void **out)
{
  return guard([&] {
    std::unique_ptr<World> w(make_world_common(d, cells, 0.0, 1, periodic, p, n_ranks, 1));
    const FaceAccess access = make_basis(w->cfg.basis, w->cfg.p).face_access;
    for (int r = 0; r < n_ranks; ++r)
      {
        w->layouts.push_back(build_dof_layout(w->mesh, w->partition, w->faces, r, w->cfg.k(), 1));
        w->plans.push_back(build_exchange_plan(w->layouts.back(), w->faces, w->partition, access,
                                               ghost_need(w->cfg.kind)));
      }
    *out = w.release();
  });
}

void dgref_world_destroy(void *w) { delete static_cast<World *>(w); }

// counts[0..7]: n_cells, n_faces, n_q_cell, n_q_face, compressed, dofs/cell,
// n_ranks, n_dofs
int dgref_world_counts(void *wp, long long *counts)
{
  return guard([&] {
    const World &w = *static_cast<World *>(wp);
    counts[0] = w.mesh.n_cells();
    counts[1] = static_cast<long long>(w.faces.size());
    counts[2] = w.geom ? w.geom->n_q_cell : 0;
    counts[3] = w.geom ? w.geom->n_q_face : 0;
    counts[4] = w.geom && w.geom->compressed() ? 1 : 0;
    counts[5] = layout_of(w, 0).dofs_per_cell;
    counts[6] = w.partition.n_ranks;
    counts[7] = counts[0] * counts[5];
  });
}

// Face list in enumerate_faces order (mesh.cpp:70-132) and ownership.
int dgref_world_faces(void *wp, std::uint32_t *interior, std::uint32_t *exterior,
                      std::uint8_t *fn_int, std::uint8_t *fn_ext,
                      int *face_owner, int *cell_owner)
{
  return guard([&] {
    const World &w = *static_cast<World *>(wp);
    for (std::size_t i = 0; i < w.faces.size(); ++i)
      {
        interior[i] = w.faces[i].interior_cell;
        exterior[i] = w.faces[i].exterior_cell;
        fn_int[i] = w.faces[i].interior_face_number;
        fn_ext[i] = w.faces[i].exterior_face_number;
        face_owner[i] = w.partition.face_owner[i];
      }
    for (int c = 0; c < w.mesh.n_cells(); ++c)
      cell_owner[c] = w.partition.cell_owner[c];
  });
}

// Geometry arrays in the reference layout (geometry.hpp:94-147).
// which: 0 inv_jac_t, 1 jxw, 2 face_jxw, 3 face_jni, 4 face_jne, 5 penalty,
// 6 cell_volume, 7 face_normal, 8 face_qpoints, 9 wq_cell, 10 wq_face
int dgref_world_geometry(void *wp, int which, double *out, long long *n)
{
  return guard([&] {
    const GeometryCache &g = *static_cast<World *>(wp)->geom;
    const std::vector<double> *v = nullptr;
    switch (which)
      {
      case 0: v = &g.inv_jac_t; break;
      case 1: v = &g.jxw; break;
      case 2: v = &g.face_jxw; break;
      case 3: v = &g.face_jni; break;
      case 4: v = &g.face_jne; break;
      case 5: v = &g.penalty; break;
      case 6: v = &g.cell_volume; break;
      case 7: v = &g.face_normal; break;
      case 8: v = &g.face_qpoints; break;
      case 9: v = &g.wq_cell; break;
      case 10: v = &g.wq_face; break;
      case 11: v = &g.coeff; break;
      default: throw std::invalid_argument("dgref_world_geometry: bad array");
      }
    if (out)
      std::memcpy(out, v->data(), sizeof(double) * v->size());
    *n = static_cast<long long>(v->size());
  });
}

// Per-rank layout (dof_layout.cpp:170-253): info[0..4] = owned_cell_begin,
// n_owned_cells, n_ghost_cells, owned_size, total_size.
int dgref_world_layout(void *wp, int rank, long long *info,
                       std::uint32_t *ghost_cells, int *ghost_owner)
{
  return guard([&] {
    const DoFLayout &l = layout_of(*static_cast<World *>(wp), rank);
    info[0] = l.owned_cell_begin;
    info[1] = l.n_owned_cells;
    info[2] = static_cast<long long>(l.ghost_global_cells.size());
    info[3] = l.owned_size;
    info[4] = l.total_size;
    if (ghost_cells)
      for (std::size_t i = 0; i < l.ghost_global_cells.size(); ++i)
        {
          ghost_cells[i] = l.ghost_global_cells[i];
          ghost_owner[i] = l.ghost_owner[i];
        }
  });
}

// Exchange plans (ghost_exchange.cpp:100-144). which: 0 send, 1 recv.
// sizes[0] = number of neighbour plans; for idx >= 0: sizes[1..3] = n_cells,
// n_offsets, n_dofs of plan idx and, if the pointers are non-null, the data.
int dgref_world_plan(void *wp, int rank, int which, int idx, int *neighbor,
                     std::uint32_t *cells, std::uint32_t *offsets,
                     std::uint32_t *dofs, long long *sizes)
{
  return guard([&] {
    const ExchangePlan &pl = static_cast<World *>(wp)->plans.at(rank);
    const auto &v = which == 0 ? pl.send : pl.recv;
    sizes[0] = static_cast<long long>(v.size());
    if (idx < 0)
      return;
    const NeighborPlan &p = v.at(idx);
    sizes[1] = static_cast<long long>(p.cells.size());
    sizes[2] = static_cast<long long>(p.dof_offsets.size());
    sizes[3] = static_cast<long long>(p.dofs.size());
    if (neighbor)
      *neighbor = p.neighbor;
    if (cells)
      std::memcpy(cells, p.cells.data(), 4 * p.cells.size());
    if (offsets)
      std::memcpy(offsets, p.dof_offsets.data(), 4 * p.dof_offsets.size());
    if (dofs)
      std::memcpy(dofs, p.dofs.data(), 4 * p.dofs.size());
  });
}

// y = A x in the canonical cell-major numbering through the reference
// RankOperator::apply. One rank: plain apply (test_operators.cpp:42-52).
// Several ranks: threaded GhostExchanger transport, exactly as
// distributed_apply (test_ghost_exchange.cpp:63-87).
int dgref_world_apply(void *wp, const double *x, double *y)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    const int nr = w.partition.n_ranks;
    const long long n = static_cast<long long>(w.mesh.n_cells()) *
                        w.ops[0]->layout().dofs_per_cell;
    const std::vector<double> xv(x, x + n);
    if (nr == 1)
      {
        GhostedVector u = w.ops[0]->layout().make_vector();
        GhostedVector yv = w.ops[0]->layout().make_vector();
        from_canonical(w.ops[0]->layout(), xv, u);
        w.ops[0]->apply(u, yv);
        std::vector<double> out;
        to_canonical(w.ops[0]->layout(), yv, out);
        std::memcpy(y, out.data(), sizeof(double) * n);
        return;
      }
    TransportHub hub(nr);
    std::vector<std::vector<double>> partial(
      nr, std::vector<double>(static_cast<std::size_t>(n), 0.0));
    run_ranks(nr, [&](int r) {
      GhostExchanger ex(w.plans[r], &w.ops[r]->layout(), &hub);
      ExchangeHooks hooks = ex.hooks();
      GhostedVector u = w.ops[r]->layout().make_vector();
      GhostedVector yv = w.ops[r]->layout().make_vector();
      from_canonical(w.ops[r]->layout(), xv, u);
      w.ops[r]->apply(u, yv, &hooks);
      to_canonical(w.ops[r]->layout(), yv, partial[r]);
    });
    for (long long i = 0; i < n; ++i)
      {
        double s = 0;
        for (int r = 0; r < nr; ++r)
          s += partial[r][i];
        y[i] = s;
      }
  });
}

// Rank-local apply on one rank with ghost values supplied in the rank's
// ghost order (for checking per-rank device results including the ghost
// region of y before compression). u_local/y_local: layout.total_size
// values in the reference W-layout of that rank.
int dgref_world_apply_rank_local(void *wp, int rank, const double *u_local,
                                 double *y_local)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    const DoFLayout &l = w.ops.at(rank)->layout();
    GhostedVector u = l.make_vector();
    GhostedVector y = l.make_vector();
    std::memcpy(u.data.data(), u_local, sizeof(double) * l.total_size);
    ExchangeHooks hooks;
    hooks.start_ghost_update = [](GhostedVector &) {};
    hooks.finish_ghost_update = [](GhostedVector &v) {
      v.state = VectorState::ghosts_valid;
    };
    hooks.compress = [](GhostedVector &) {};
    u.state = VectorState::ghosts_valid;
    w.ops[rank]->apply(u, y, &hooks);
    std::memcpy(y_local, y.data.data(), sizeof(double) * l.total_size);
  });
}

// RankOperator::assemble_rhs of one rank (operators.cpp:266-282), rank-local
// layout (W = 1 worlds: owned cells then ghosts).
int dgref_world_rhs(void *wp, int rank, double *rhs_local)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    const DoFLayout &l = w.ops.at(rank)->layout();
    GhostedVector r = l.make_vector();
    w.ops[rank]->assemble_rhs(r);
    std::memcpy(rhs_local, r.data.data(), sizeof(double) * l.total_size);
  });
}

// Dense assembled oracle (oracle.cpp:205-426), <= 20000 dofs, column-major
// n x n written row-major into out.
int dgref_world_assemble(void *wp, double *out)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    if (w.external_geometry)
      throw std::invalid_argument(
        "dgref_world_assemble: the dense oracle recomputes geometry from "
        "the reference mesh; not available for injected geometry");
    const Eigen::MatrixXd a = oracle::assemble_operator(w.cfg, w.mesh);
    const Eigen::Index n = a.rows();
    for (Eigen::Index i = 0; i < n; ++i)
      for (Eigen::Index j = 0; j < n; ++j)
        out[i * n + j] = a(i, j);
  });
}

// Wall seconds for n_applies applications, all ranks in lockstep over the
// threaded transport; BenchWorld::run (bench.cpp:128-166) verbatim in
// behaviour (input fill 0.25 + 1e-4 (i mod 97)).
int dgref_world_time(void *wp, long long n_applies, double *seconds)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    using Clock = std::chrono::steady_clock;
    const int nr = static_cast<int>(w.ops.size());
    if (nr == 1)
      {
        GhostedVector u = w.ops[0]->layout().make_vector();
        GhostedVector y = w.ops[0]->layout().make_vector();
        for (std::size_t i = 0; i < u.data.size(); ++i)
          u.data[i] = 0.25 + 1e-4 * static_cast<double>(i % 97);
        const auto t0 = Clock::now();
        for (long long i = 0; i < n_applies; ++i)
          {
            u.state = VectorState::clean;
            w.ops[0]->apply(u, y);
          }
        *seconds = std::chrono::duration<double>(Clock::now() - t0).count();
        return;
      }
    TransportHub hub(nr);
    const auto t0 = Clock::now();
    run_ranks(nr, [&](int r) {
      GhostExchanger ex(w.plans[r], &w.ops[r]->layout(), &hub);
      ExchangeHooks hooks = ex.hooks();
      GhostedVector u = w.ops[r]->layout().make_vector();
      GhostedVector y = w.ops[r]->layout().make_vector();
      for (std::size_t i = 0; i < u.data.size(); ++i)
        u.data[i] = 0.25 + 1e-4 * static_cast<double>(i % 97);
      for (long long i = 0; i < n_applies; ++i)
        {
          u.state = VectorState::clean;
          w.ops[r]->apply(u, y, &hooks);
        }
    });
    *seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  });
}

// conjugate_gradient(make_apply(op), b, x, tol, maxit) on rank 0 of a
// single-rank world (solvers.cpp:24-68,189-206); canonical b, x.
int dgref_world_cg(void *wp, const double *b, double *x, double rel_tol, int max_iterations,
                   int *converged, int *iterations, double *relative_residual)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    if (w.ops.size() != 1)
      throw std::invalid_argument("dgref_world_cg: single-rank worlds only");
    const long long n = w.ops[0]->layout().owned_size;
    const std::vector<double> bv(b, b + n);
    std::vector<double> xv;
    const SolveReport r = conjugate_gradient(make_apply(*w.ops[0]), bv, xv, rel_tol,
                                             max_iterations);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *converged = r.converged ? 1 : 0;
    *iterations = r.iterations;
    *relative_residual = r.relative_residual;
  });
}

// Instrumented flop count of one application (counters x W, bench.cpp:339).
int dgref_world_flops(void *wp, double *flops)
{
  return guard([&] {
    World &w = *static_cast<World *>(wp);
    const int nr = static_cast<int>(w.ops.size());
    for (auto &op : w.ops)
      op->reset_counters();
    double tmp;
    dgref_world_time(wp, 1, &tmp);
    double f = 0;
    for (auto &op : w.ops)
      f += static_cast<double>(op->counters().flops());
    *flops = f * w.cfg.W;
    (void)nr;
  });
}

} // extern "C"
