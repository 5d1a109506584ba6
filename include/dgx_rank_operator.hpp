// Reference-side drop-in: a sibling of dg::RankOperator (proj/include/dg/
// operators.hpp:69-106) with the identical constructor and apply() semantics,
// executing on a B200 through include/dgx.h. Header-only; it is compiled in
// the reference's tree (needs <dg/...>) and linked against libdgx.so.
//
//   dgx_ref::RankOperator op(mesh, partition, faces, geometry, cfg, rank);
//   op.apply(u, y, &hooks);   // same GhostedVector state machine
//
// Vectors stay the reference's host GhostedVectors; each apply copies u
// (owned + ghosts) to the device and y back (use the C ABI with device
// pointers directly to keep vectors resident). The layout is the reference
// layout with W = 1 (lane batching is a CPU SIMD artefact; cfg.W is
// accepted and ignored). Exchange hooks are the reference's own: the ghost
// update completes on the host before the device apply, compress runs after.
#pragma once

#include <dg/dof_layout.hpp>
#include <dg/geometry.hpp>
#include <dg/mesh.hpp>
#include <dg/operators.hpp>

#include <dgx.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace dgx_ref
{

inline void check(dgx_status s)
{
  switch (s)
    {
    case DGX_OK:
      return;
    case DGX_INVALID_ARGUMENT:
      throw std::invalid_argument(dgx_last_error());
    case DGX_LOGIC_ERROR:
      throw std::logic_error(dgx_last_error());
    default:
      throw std::runtime_error(dgx_last_error());
    }
}

class RankOperator
{
public:
  RankOperator(const dg::Mesh &mesh, const dg::Partition &partition,
               const std::vector<dg::RawFace> &faces,
               std::shared_ptr<const dg::GeometryCache> geometry,
               const dg::OperatorConfig &config, int rank, int device = 0)
    : cfg_(config), geom_(std::move(geometry))
  {
    if (config.kind != dg::OperatorKind::laplacian &&
        config.kind != dg::OperatorKind::advection)
      throw std::invalid_argument("dgx_ref::RankOperator: Laplacian or advection only");
    if (config.kind == dg::OperatorKind::advection && !config.velocity.is_constant())
      throw std::invalid_argument(
        "dgx_ref::RankOperator: pass a variable velocity through dgx_set_velocity");
    if (mesh.d != config.d)
      throw std::invalid_argument("RankOperator: mesh dimension mismatch");
    if (!geom_ || geom_->k != config.k() || geom_->l != config.k() ||
        geom_->equation != config.equation() ||
        geom_->variant != dg::GeometryVariant::g3)
      throw std::invalid_argument(
        "RankOperator: geometry cache does not match the configuration");
    static_assert(sizeof(dg::RawFace) == sizeof(dgx_raw_face), "RawFace layout");

    dgx_setup s{};
    s.mesh.d = mesh.d;
    for (int a = 0; a < 3; ++a)
      {
        s.mesh.cells_per_dim[a] = mesh.cells_per_dim[a];
        s.mesh.lo[a] = mesh.lo[a];
        s.mesh.hi[a] = mesh.hi[a];
        s.mesh.periodic[a] = mesh.boundary[2 * a].periodic ? 1 : 0;
      }
    for (int b = 0; b < 6; ++b)
      s.mesh.dirichlet_id[b] = mesh.boundary[b].dirichlet_id;
    s.mesh.deform_amplitude = mesh.deform_amplitude;
    s.mesh.mapping_degree = mesh.mapping_degree;
    s.faces = reinterpret_cast<const dgx_raw_face *>(faces.data());
    s.n_faces = static_cast<int64_t>(faces.size());
    s.n_ranks = partition.n_ranks;
    ranges_.resize(2 * partition.n_ranks);
    for (int r = 0; r < partition.n_ranks; ++r)
      {
        ranges_[2 * r] = partition.rank_cell_range[r].first;
        ranges_[2 * r + 1] = partition.rank_cell_range[r].second;
      }
    s.cell_owner = partition.cell_owner.data();
    s.rank_cell_range = ranges_.data();
    s.face_owner = partition.face_owner.data();
    s.rank = rank;
    s.config.d = config.d;
    s.config.p = config.p;
    s.config.W = 1;
    s.config.basis = static_cast<int>(config.basis); // BasisKind order (basis.hpp:10-15)
    s.config.geometry_variant = 3;
    s.config.precision = 0;
    s.config.kind = config.kind == dg::OperatorKind::advection ? 1 : 0;
    for (int a = 0; a < 3; ++a)
      s.config.velocity[a] = config.velocity.constant[a];
    s.geometry.source = DGX_GEOMETRY_HOST_ARRAYS;
    s.geometry.compressed = geom_->compressed() ? 1 : 0;
    s.geometry.inv_jac_t = geom_->inv_jac_t.data();
    s.geometry.jxw = geom_->jxw.data();
    s.geometry.face_jxw = geom_->face_jxw.data();
    s.geometry.face_jni = geom_->face_jni.data();
    s.geometry.face_jne = geom_->face_jne.data();
    s.geometry.penalty = geom_->penalty.data();
    s.geometry.face_normal = geom_->face_normal.data();
    check(dgx_create(&s, device, &op_));
    layout_ = dg::build_dof_layout(mesh, partition, faces, rank, config.k(), 1);
  }

  ~RankOperator()
  {
    if (op_)
      dgx_destroy(op_);
  }
  RankOperator(const RankOperator &) = delete;
  RankOperator &operator=(const RankOperator &) = delete;

  const dg::DoFLayout &layout() const { return layout_; }
  const dg::OperatorConfig &config() const { return cfg_; }

  // y = A u with the reference's state machine (operators.cpp:217-264).
  void apply(dg::GhostedVector &u, dg::GhostedVector &y,
             const dg::ExchangeHooks *hooks = nullptr)
  {
    if (u.data.size() != static_cast<std::size_t>(layout_.total_size) ||
        y.data.size() != static_cast<std::size_t>(layout_.total_size))
      throw std::invalid_argument("apply: vector size mismatch");
    const bool have_ghosts = !layout_.ghost_global_cells.empty();
    if (hooks && hooks->start_ghost_update)
      hooks->start_ghost_update(u);
    else if (have_ghosts)
      throw std::logic_error(
        "apply: layout has ghost cells but no exchange hooks were given");
    else
      u.state = dg::VectorState::ghosts_valid;
    if (have_ghosts && u.state != dg::VectorState::ghosts_valid)
      {
        if (hooks && hooks->finish_ghost_update)
          hooks->finish_ghost_update(u);
        else
          throw std::logic_error(
            "apply: ghost-coupled face reached without a way to finish the "
            "ghost update");
      }
    check(dgx_apply_host(op_, u.data.data(), y.data.data()));
    if (have_ghosts)
      y.state = dg::VectorState::has_remote_contributions;
    if (hooks && hooks->compress)
      hooks->compress(y);
    else
      y.state = dg::VectorState::clean;
  }

private:
  dg::OperatorConfig cfg_;
  std::shared_ptr<const dg::GeometryCache> geom_;
  dg::DoFLayout layout_;
  std::vector<int> ranges_;
  dgx_op *op_ = nullptr;
};

} // namespace dgx_ref
